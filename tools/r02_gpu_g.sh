# Round-2 GPU call G (4 GPUs): the final defaults (u = 1 MiB, 64-CTA-per-SM snapshot pack,
# rebuild shares for m >= 3, progressive HAS issue) -- single-GPU suite and the ncu of the
# new pack grid side by side, the multi-GPU suite at 4 GPUs, bench lines at N = 4, 2, 1,
# NVLink counters of the m = 4 encode with u = 1 MiB, the C5 drill at m = 4.
set -x
(CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -v -rs --durations=15 -k "not every_tuning_knob" > gpurun_out/r02g_pytest_gpu_1.log 2>&1) &
(CUDA_VISIBLE_DEVICES=1 timeout 900 bash tools/ncu_profile.sh r02_tma64 pack_all_tma 2 2 > gpurun_out/r02g_ncu_pack.log 2>&1) &
wait
timeout 1500 python -m pytest tests/test_multigpu.py -m gpu -v -rs --durations=10 > gpurun_out/r02g_pytest_multigpu_4gpu.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 > gpurun_out/r02g_bench_n4.jsonl 2> gpurun_out/r02g_bench_n4.err
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/r02g_bench_n2.jsonl 2> gpurun_out/r02g_bench_n2.err
timeout 600 python bench.py > gpurun_out/r02g_bench_n1.jsonl 2> gpurun_out/r02g_bench_n1.err
X="python tools/xor_local2.py --m 4 --bucket 1073741824 --reps 1"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum --clock-control none -k regex:xor_tma -c 8 --csv --log-file gpurun_out/r02g_xortma_m4_nvlink.csv $X > gpurun_out/r02g_ncu_xor_m4_metrics.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29700 --nproc-per-node 4 tools/sweep.py --config c5_13b_drill --buckets 1024 --n-slots 0 --reps 1 --drill --lost 0,3 > gpurun_out/r02g_c5_drill_m4.jsonl 2> gpurun_out/r02g_c5_drill_m4.err
ls -la gpurun_out | grep r02g
