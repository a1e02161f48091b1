export CKPT_TIMEOUT_S=60
port=29760
for i in 1 2; do
  for L in new legacy; do
    port=$((port+1))
    if [ $L = legacy ]; then export CKPT_WAIT_LEGACY=1; else unset CKPT_WAIT_LEGACY; fi
    timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port tools/sweep.py --config c1_16mb_fp32_m8 --buckets 16 --n-slots 0 --reps 30 2>&1 | grep '^{"config' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$L', d['snapshot_ms'], d['pack_us_per_launch'], d['xor_us_per_launch'])"
  done
done
