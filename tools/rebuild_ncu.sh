#!/bin/bash
# ncu evidence for the rebuild (Eq 2) on the XOR kernel: one process, m GPUs (LOCAL group),
# lose member 1, survivors rebuild it from their device images (P2P stores over NVLink).
set -u
M=${1:-2}
mkdir -p gpurun_out
CMD="python tools/xor_local2.py --m $M --bucket 1073741824 --reps 1 --rebuild 1"
$CMD > gpurun_out/rebuild_plain.log 2>&1 || { echo plain failed; tail -5 gpurun_out/rebuild_plain.log; exit 1; }
tail -1 gpurun_out/rebuild_plain.log
# the encode launches come first (one per member and snapshot): skip them, keep the rebuild's
ncu --metrics nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:xor_tma -s $((2 * M)) -c 8 --csv $CMD > gpurun_out/rebuild_ncu.csv 2>&1; echo "ncu rc=$?"
grep -E '"(nvl|gpu__time|dram)' gpurun_out/rebuild_ncu.csv | cut -d, -f1,5,10,13,15 | head -40
