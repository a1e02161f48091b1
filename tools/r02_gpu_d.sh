# Round-2 GPU call D (2 GPUs): the whole GPU suite at HEAD (single-GPU tests + multi-GPU at 2),
# HAS 1F1B on a real 2-stage pipeline, N=1 co-run A/B (pack SM budget, L2 evict_first),
# the m = 2 stripe-unit A/B of the encode.
set -x
timeout 2400 python -m pytest tests -m gpu -v -rs --durations=20 > gpurun_out/r02d_pytest_gpu_all_2gpu.log 2>&1
timeout 420 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29577 tools/has_1f1b.py --watchdog-s 360 --out gpurun_out/r02d_has_1f1b.jsonl > gpurun_out/r02d_has_1f1b.log 2>&1
B="python bench.py --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/r02d_corun_default.jsonl 2>&1
timeout 600 $B --max-ctas 64 > gpurun_out/r02d_corun_ctas64.jsonl 2>&1
CKPT_PACK_L2HINT=1 timeout 600 $B > gpurun_out/r02d_corun_l2hint.jsonl 2>&1
CKPT_PACK_L2HINT=1 timeout 600 $B --max-ctas 64 > gpurun_out/r02d_corun_l2hint_ctas64.jsonl 2>&1
timeout 600 $B --max-ctas 32 > gpurun_out/r02d_corun_ctas32.jsonl 2>&1
for u in 4096 16384 65536 262144; do timeout 300 python tools/xor_local2.py --m 2 --reps 3 --unit $u >> gpurun_out/r02d_unit_m2.jsonl 2>>gpurun_out/r02d_unit_m2.err; done
ls -la gpurun_out | grep r02d
