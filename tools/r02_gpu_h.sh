# Round-2 GPU call H (1 GPU): the tuning-knob subprocess tests at the final defaults, the
# smoke entry point, and which copy-engine traffic slows the co-running GEMM.
set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -v -rs -k "every_tuning_knob or windowed or c2_bench_config" > gpurun_out/r02h_pytest_knobs_1.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02h_smoke.log 2>&1
timeout 900 python tools/gemm_vs_copy.py > gpurun_out/r02h_gemm_vs_copy.jsonl 2> gpurun_out/r02h_gemm_vs_copy.err
ls -la gpurun_out | grep r02h
