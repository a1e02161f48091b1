# Round-2 GPU call C (4 GPUs): CE mirror parity + elastic drill diagnostics, HAS 1F1B with a
# watchdog, the m=2 CE-mirror A/B, bench lines at N = 1, 2, 4, ncu of the N=1 pack and of the
# m = 4 XOR encode (NVLink counters + --set full), the m = 4 rebuild-shares A/B, fabric probes.
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rs -k "drill_rebuild_every_rank or encode_matches_oracle" > gpurun_out/r02c_pytest_ce_mirror_1.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 600 python -m pytest tests/test_multigpu.py -m gpu -v -rs -k "elastic or full_image" > gpurun_out/r02c_pytest_elastic_full_2gpu.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 420 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29577 tools/has_1f1b.py --watchdog-s 360 --out gpurun_out/r02c_has_1f1b.jsonl > gpurun_out/r02c_has_1f1b.log 2>&1
for fl in 0 16; do timeout 300 python tools/xor_local2.py --m 2 --reps 3 --flags $fl >> gpurun_out/r02c_mirror_ab.jsonl 2>>gpurun_out/r02c_mirror_ab.err; done
timeout 600 python bench.py > gpurun_out/r02c_bench_n1.jsonl 2> gpurun_out/r02c_bench_n1.err
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/r02c_bench_n2.jsonl 2> gpurun_out/r02c_bench_n2.err
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --gather ce > gpurun_out/r02c_bench_n2_mirror.jsonl 2> gpurun_out/r02c_bench_n2_mirror.err
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 > gpurun_out/r02c_bench_n4.jsonl 2> gpurun_out/r02c_bench_n4.err
timeout 900 bash tools/ncu_profile.sh r02_tma8 pack_all_tma 2 2 > gpurun_out/r02c_ncu_pack.log 2>&1
X="python tools/xor_local2.py --m 4 --bucket 1073741824 --reps 1"
timeout 300 $X > gpurun_out/r02c_xor_m4_plain.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum --clock-control none -k regex:xor_tma -c 8 --csv --log-file gpurun_out/r02c_xortma_m4_nvlink.csv $X > gpurun_out/r02c_ncu_xor_m4_metrics.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'pack|xor' -c 200 --csv --log-file gpurun_out/r02c_xortma_m4_launches.csv $X > gpurun_out/r02c_ncu_xor_m4_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:xor_tma -s 4 -c 1 -o gpurun_out/prof_r02_xortma_m4 $X > gpurun_out/r02c_ncu_xor_m4_full.log 2>&1
N=4 CFG=c5_13b_drill LOST=0,3 timeout 1200 bash tools/rb_share_ab.sh > gpurun_out/r02c_rb_share_ab_m4.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/fabric tools/fabric_probe.cu
for mode in sm_pull xorpat4k xorpat16k; do for c in 32 64; do timeout 60 /tmp/fabric 4 1536 $mode $c 5 >> gpurun_out/r02c_fabric.jsonl 2>>gpurun_out/r02c_fabric.err; done; done
ls -la gpurun_out
