# Round-2 GPU call F (4 GPUs): stripe-unit A/B of the encode at m = 4 and 3 (large units and
# u = 0, the paper's whole-shard split), then, concurrently on separate GPUs, the snapshot
# pack's grid (CTAs per SM) A/B at N = 1 and the C3 CTA-budget sweep with the GEMM co-run.
set -x
for u in 262144 1048576 4194304 0; do timeout 300 python tools/xor_local2.py --m 4 --reps 3 --unit $u >> gpurun_out/r02f_unit_m4.jsonl 2>>gpurun_out/r02f_unit_m4.err; done
for u in 65536 262144 1048576 0; do CUDA_VISIBLE_DEVICES=0,1,2 timeout 300 python tools/xor_local2.py --m 3 --reps 3 --unit $u >> gpurun_out/r02f_unit_m3.jsonl 2>>gpurun_out/r02f_unit_m3.err; done
(for w in 8 16 32 64; do CUDA_VISIBLE_DEVICES=0 CKPT_PACK_WAVES=$w timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r02f_waves$w.jsonl 2>&1; done) &
(CUDA_VISIBLE_DEVICES=1 timeout 1500 python tools/sweep.py --config c3_13b_tp4pp2 --buckets 64 --n-slots 4 --flags 2 --max-ctas 1,2,4,8,16,0 --corun --reps 2 > gpurun_out/r02f_c3_ctas.jsonl 2> gpurun_out/r02f_c3_ctas.err) &
wait
ls -la gpurun_out | grep r02f
