# Round-2 GPU call N (2 GPUs): why the pack is slower at N >= 2 -- the same two processes
# as one m = 2 group (IPC) vs as two m = 1 groups.
set -x
R="python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="bench.py --gpus 2 --no-corun --no-e2e --no-cpu-baseline"
timeout 600 $R --master-port 29621 $B > gpurun_out/r02n_n2_m2.jsonl 2> gpurun_out/r02n_n2_m2.err
timeout 600 $R --master-port 29622 $B --group-size 1 > gpurun_out/r02n_n2_m1.jsonl 2> gpurun_out/r02n_n2_m1.err
timeout 600 $R --master-port 29623 $B --device-only > gpurun_out/r02n_n2_m2_dev.jsonl 2> gpurun_out/r02n_n2_m2_dev.err
ls -la gpurun_out | grep r02n
