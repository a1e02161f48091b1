# Round-2 GPU call L (4 GPUs): the multi-GPU suite at the final HEAD, then SURVEY 8(d)'s
# per-config measurements at m = 4 with the final defaults: C3 bucket x CTA-budget sweep
# with the GEMM co-run (ring staging), C4 (the paper's shape) with a drill, C1 (latency).
set -x
timeout 1500 python -m pytest tests/test_multigpu.py -m gpu -v -rs --durations=10 > gpurun_out/r02l_pytest_multigpu_4gpu.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
timeout 1200 $R --master-port 29701 tools/sweep.py --config c3_13b_tp4pp2 --buckets 4,64,512 --n-slots 4 --flags 2 --max-ctas 4,0 --corun --corun-pairs 6 --reps 2 > gpurun_out/r02l_c3_m4.jsonl 2> gpurun_out/r02l_c3_m4.err
timeout 900 $R --master-port 29702 tools/sweep.py --config c4_34b_tp8_stage0 --buckets 512 --n-slots 0 --reps 2 --drill --lost 0,3 > gpurun_out/r02l_c4_m4.jsonl 2> gpurun_out/r02l_c4_m4.err
timeout 600 $R --master-port 29703 tools/sweep.py --config c1_16mb_fp32_m8 --unit 65536 --buckets 64 --n-slots 0 --reps 5 --drill --lost 0,3 > gpurun_out/r02l_c1_m4.jsonl 2> gpurun_out/r02l_c1_m4.err
ls -la gpurun_out | grep r02l
