#!/bin/bash
# A/B of who re-encodes the lost member's parity row during a rebuild: the survivors in
# shares (CKPT_OPT_REBUILD_SHARES, reading Q27) vs the lost member itself (default);
# m = number of GPUs (N), C2 7B/TP8 state, drills losing rank 0 and rank 1.
mkdir -p gpurun_out
N=${N:-2}
CFG=${CFG:-c2_7b_tp8}
for mode in shares self; do
  fl=2048; [ $mode = shares ] && fl=512  # CKPT_OPT_REBUILD_SELF / CKPT_OPT_REBUILD_SHARES
  timeout 400 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 \
    --master-port $((29700 + fl % 7)) --nproc-per-node $N tools/sweep.py --config $CFG --buckets 1024 --n-slots 0 \
    --reps 1 --drill --lost ${LOST:-0,1} --flags $fl > gpurun_out/sw_rb_ab_m${N}_$mode.jsonl 2> gpurun_out/sw_rb_ab_m${N}_$mode.err
  echo "$mode rc=$?"
  python -c "
import json
for l in open('gpurun_out/sw_rb_ab_m${N}_$mode.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print([(x['lost'],x['rebuild_ms'],x['bit_exact_all_bytes'],x['rank0_rebuild_kernel_gbs']) for x in d.get('drill',[])])
"
done
