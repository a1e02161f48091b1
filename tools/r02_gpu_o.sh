# Round-2 GPU call O (1 GPU): after removing the L2-hint branch from the pack kernel -- the
# pack/load parity tests, smoke, and the N=1 bench line without the co-run.
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rs -k "snapshot_unprotected or c2_bench_config or no_writes_outside or load_from_device or group_encode or drill_rebuild" > gpurun_out/r02o_pytest_pack_1.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02o_smoke.log 2>&1
timeout 600 python bench.py --no-corun > gpurun_out/r02o_bench_n1.jsonl 2> gpurun_out/r02o_bench_n1.err
ls -la gpurun_out | grep r02o
