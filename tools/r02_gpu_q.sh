# Round-2 GPU call Q (4 GPUs): the N = 4 bench line at HEAD with the three co-run
# configurations (8 ABBA pairs each to fit the remaining budget).
set -x
timeout 1000 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641 bench.py --gpus 4 --corun-pairs 8 > gpurun_out/r02q_bench_n4.jsonl 2> gpurun_out/r02q_bench_n4.err
ls -la gpurun_out | grep r02q
