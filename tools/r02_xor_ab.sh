# A/B of the parity encode at m = 2 and 4 (one process drives m GPUs, DEVICE_ONLY):
# pull XOR tile configurations, CTA budgets, and the push-mode encode.
set -x
out=gpurun_out/r02_xor_ab.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rs -k "push or has_three or full_image" > gpurun_out/r02_pytest_push_1.log 2>&1
for m in 4 2; do
  for tile in 0 1 2; do
    for ctas in 0 128; do
      if [ $ctas = 0 ]; then unset CKPT_XOR_CTAS; else export CKPT_XOR_CTAS=$ctas; fi
      echo "{\"m\": $m, \"tile\": $tile, \"xor_ctas_env\": $ctas}" >> $out
      CKPT_XOR_TILE=$tile timeout 300 python tools/xor_local2.py --m $m --reps 3 >> $out 2>>gpurun_out/r02_xor_ab.err
    done
  done
  unset CKPT_XOR_CTAS
  for ctas in 0 64 128 296; do
    if [ $ctas = 0 ]; then unset CKPT_XOR_CTAS; else export CKPT_XOR_CTAS=$ctas; fi
    echo "{\"m\": $m, \"push\": 1, \"xor_ctas_env\": $ctas}" >> $out
    timeout 300 python tools/xor_local2.py --m $m --reps 3 --flags 1024 >> $out 2>>gpurun_out/r02_xor_ab.err
  done
  unset CKPT_XOR_CTAS
done
