# Round-2 GPU call J (1 GPU): what in a snapshot costs the co-running GEMM (tools/corun_probe.py).
set -x
timeout 1500 python tools/corun_probe.py --pairs 10 > gpurun_out/r02j_corun_probe.jsonl 2> gpurun_out/r02j_corun_probe.err
ls -la gpurun_out | grep r02j
