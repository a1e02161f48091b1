mkdir -p gpurun_out
timeout 150 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "test_group_drill_rebuild_every_rank or test_device_only_drill or test_arc_schemes_snapshot_and_every_recovery" > gpurun_out/rb_t1.log 2>&1; r1=$?; echo t1=$r1; tail -2 gpurun_out/rb_t1.log
[ $r1 = 0 ] || exit 11
timeout 150 python -m pytest tests/test_multigpu.py -m gpu -x -q -k "test_ipc_group_all_gpus and (case0 or case1)" > gpurun_out/rb_t2.log 2>&1; r2=$?; echo t2=$r2; tail -2 gpurun_out/rb_t2.log
[ $r2 = 0 ] || exit 12
timeout 150 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29611 --nproc-per-node 4 tools/sweep.py --config c5_13b_drill --buckets 1024 --n-slots 0 --reps 1 --drill --lost 0,3 --flags 512 > gpurun_out/sw_c5_m4_share.jsonl 2> gpurun_out/sw_c5_m4_share.err; echo c5=$?
python - <<'PY'
import json
for l in open("gpurun_out/sw_c5_m4_share.jsonl"):
    if l.startswith("{"):
        d=json.loads(l); print([(x["lost"],x["rebuild_ms"],x["load_ms"],x["bit_exact_sampled"]) for x in d.get("drill",[])])
PY
