# Round-2 GPU call B (4 GPUs): bench lines at N = 1, 2, 4 (torchrun), the ncu launch list +
# --set full capture of the N=1 pack, and the NVLink counters + --set full capture of the
# m = 4 XOR encode (one process drives 4 GPUs: tools/xor_local2.py).
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/fabric tools/fabric_probe.cu
for mode in sm_pull xorpat4k xorpat16k; do for c in 32 64; do timeout 60 /tmp/fabric 4 1536 $mode $c 5 >> gpurun_out/r02_fabric_b.jsonl 2>>gpurun_out/r02_fabric_b.err; done; done
for c in 16 32; do CKPT_XOR_CTAS=$c timeout 300 python tools/xor_local2.py --m 4 --reps 3 >> gpurun_out/r02_xor_fewctas.jsonl 2>>gpurun_out/r02_xor_fewctas.err; done
timeout 600 python bench.py > gpurun_out/r02_bench_n1.jsonl 2> gpurun_out/r02_bench_n1.err
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/r02_bench_n2.jsonl 2> gpurun_out/r02_bench_n2.err
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 > gpurun_out/r02_bench_n4.jsonl 2> gpurun_out/r02_bench_n4.err
timeout 900 bash tools/ncu_profile.sh r02_tma8 pack_all_tma 2 2 > gpurun_out/r02_ncu_pack.log 2>&1
X="python tools/xor_local2.py --m 4 --bucket 1073741824 --reps 1"
timeout 300 $X > gpurun_out/r02_xor_m4_plain.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum --clock-control none -k regex:xor_tma -c 8 --csv --log-file gpurun_out/r02_xortma_m4_nvlink.csv $X > gpurun_out/r02_ncu_xor_m4_metrics.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'pack|xor' -c 200 --csv --log-file gpurun_out/r02_xortma_m4_launches.csv $X > gpurun_out/r02_ncu_xor_m4_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:xor_tma -s 4 -c 1 -o gpurun_out/prof_r02_xortma_m4 $X > gpurun_out/r02_ncu_xor_m4_full.log 2>&1
N=4 CFG=c5_13b_drill LOST=0,3 timeout 1200 bash tools/rb_share_ab.sh > gpurun_out/r02_rb_share_ab_m4.log 2>&1
ls -la gpurun_out
