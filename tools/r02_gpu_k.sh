# Round-2 GPU call K (1 GPU): the final HEAD -- whole single-GPU suite (incl. the knob
# subprocess tests), smoke, and the driver's default bench line (with the C4 paper shape).
set -x
timeout 600 python bench.py > gpurun_out/r02k_bench_n1.jsonl 2> gpurun_out/r02k_bench_n1.err
timeout 1800 python -m pytest tests -m gpu -v -rs --durations=15 > gpurun_out/r02k_pytest_gpu_1.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02k_smoke.log 2>&1
ls -la gpurun_out | grep r02k
