# Round-2 GPU call T (1 GPU): the driver's default bench command at the final HEAD.
set -x
timeout 700 python bench.py > gpurun_out/r02t_bench_n1.jsonl 2> gpurun_out/r02t_bench_n1.err
