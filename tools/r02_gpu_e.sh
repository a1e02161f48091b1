# Round-2 GPU call E (4 GPUs): the changed paths (windowed gated issue, shares default, knob
# L2 hint, CE mirror) on one GPU, the multi-GPU suite at 4 GPUs (shares default over IPC,
# elastic drill with per-attempt store prefix), the m = 4 stripe-unit A/B of the encode,
# final bench lines at N = 1, 2, 4 (co-run with NVML clock/power per window).
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -v -rs -k "windowed or drill_rebuild_every_rank or flag_must_agree or has_ or L2HINT or fence" > gpurun_out/r02e_pytest_changed_1.log 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -m gpu -v -rs --durations=10 > gpurun_out/r02e_pytest_multigpu_4gpu.log 2>&1
for u in 4096 16384 65536 262144; do timeout 300 python tools/xor_local2.py --m 4 --reps 3 --unit $u >> gpurun_out/r02e_unit_m4.jsonl 2>>gpurun_out/r02e_unit_m4.err; done
timeout 600 python bench.py > gpurun_out/r02e_bench_n1.jsonl 2> gpurun_out/r02e_bench_n1.err
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/r02e_bench_n2.jsonl 2> gpurun_out/r02e_bench_n2.err
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 > gpurun_out/r02e_bench_n4.jsonl 2> gpurun_out/r02e_bench_n4.err
ls -la gpurun_out | grep r02e
