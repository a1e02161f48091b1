# Round-2 GPU call R (1 GPU): the whole single-GPU suite and smoke at the final HEAD.
set -x
timeout 1100 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/r02r_pytest_gpu_1.log 2>&1
timeout 200 python __graft_entry__.py smoke > gpurun_out/r02r_smoke.log 2>&1
ls -la gpurun_out | grep r02r
