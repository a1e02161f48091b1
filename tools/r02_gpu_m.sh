# Round-2 GPU call M (2 GPUs): final bench lines at N = 1 and 2 with the third co-run
# configuration (ring of 4 small slots).
set -x
timeout 900 python bench.py > gpurun_out/r02m_bench_n1.jsonl 2> gpurun_out/r02m_bench_n1.err
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/r02m_bench_n2.jsonl 2> gpurun_out/r02m_bench_n2.err
ls -la gpurun_out | grep r02m
