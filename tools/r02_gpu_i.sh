# Round-2 GPU call I (1 GPU): a tighter co-run estimate -- the bench's co-run with 40 ABBA
# pairs per configuration, and the raw copy-engine traffic experiment with 20 pairs.
set -x
timeout 900 python bench.py --no-e2e --no-cpu-baseline --corun-pairs 40 > gpurun_out/r02i_corun40.jsonl 2> gpurun_out/r02i_corun40.err
timeout 900 python tools/gemm_vs_copy.py --pairs 20 > gpurun_out/r02i_gemm_vs_copy20.jsonl 2> gpurun_out/r02i_gemm_vs_copy20.err
ls -la gpurun_out | grep r02i
