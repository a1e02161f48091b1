#!/bin/bash
# SURVEY.md 8(d) configs on a 4-GPU box (C4 at 1/2/4 GPUs, C1 and C3/C5 at m=4).
# Every multi-rank run is bounded by `timeout`; results: gpurun_out/sw_*.jsonl
export CKPT_TIMEOUT_S=120
mkdir -p gpurun_out
TR="timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P=29600
run() { local tag=$1; shift; P=$((P+1)); echo "== $tag"; "$@" > gpurun_out/sw_$tag.jsonl 2> gpurun_out/sw_$tag.err; echo "rc=$?"; grep -c config gpurun_out/sw_$tag.jsonl; }
run c1_m4_host  $TR --nproc-per-node 4 --master-port $P tools/sweep.py --config c1_16mb_fp32_m8 --buckets 16 --n-slots 0 --reps 9 --drill
run c1_m4_dev   $TR --nproc-per-node 4 --master-port $((P+50)) tools/sweep.py --config c1_16mb_fp32_m8 --buckets 16 --device-only --reps 9 --drill
run c4_m1       timeout 600 python tools/sweep.py --config c4_34b_tp8_stage0 --buckets 1024 --n-slots 0 --reps 3
run c4_m2       $TR --nproc-per-node 2 --master-port $((P+60)) tools/sweep.py --config c4_34b_tp8_stage0 --buckets 1024 --n-slots 0 --reps 3 --drill --lost 1
run c4_m4       $TR --nproc-per-node 4 --master-port $((P+70)) tools/sweep.py --config c4_34b_tp8_stage0 --buckets 1024 --n-slots 0 --reps 3 --drill --lost 0,3
run c3_ring_m4  $TR --nproc-per-node 4 --master-port $((P+80)) tools/sweep.py --config c3_13b_tp4pp2 --buckets 4,16,64,256,512 --n-slots 4 --reps 2
run c5_m4       $TR --nproc-per-node 4 --master-port $((P+90)) tools/sweep.py --config c5_13b_drill --buckets 1024 --n-slots 0 --reps 2 --drill --lost 0,1,2,3
