set -u
mkdir -p gpurun_out
CMD="python tools/xor_local2.py --m 2 --bucket 1073741824 --reps 2"
$CMD > gpurun_out/xortma_plain.log 2>&1 || { echo plain failed; tail -5 gpurun_out/xortma_plain.log; exit 1; }
tail -1 gpurun_out/xortma_plain.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'pack|xor|signal' -c 200 --csv --log-file gpurun_out/launches_r01_xortma.csv $CMD > gpurun_out/ncu_launch_xortma.log 2>&1; echo "launch rc=$?"
ncu --set full --clock-control none --import-source on -k regex:xor_tma -s 1 -c 2 -o gpurun_out/prof_r01_xortma $CMD > gpurun_out/ncu_full_xortma.log 2>&1; echo "full rc=$?"
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/b2_final.log 2>&1; echo "bench rc=$?"; grep metric gpurun_out/b2_final.log | cut -c1-300
