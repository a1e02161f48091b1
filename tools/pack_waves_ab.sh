# A/B: persistent TMA pack (1 CTA per SM) vs short-lived CTAs (k per SM) -- pack rate and
# the co-running GEMM's slowdown at N=1 (bench.py, kernel path)
for w in ${WAVES:-1 8 64}; do
  CKPT_PACK_WAVES=$w timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{"metric' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('waves', $w, d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d['gemm_corun']['this_config']['slowdown_pct'])"
done
