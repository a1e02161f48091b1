set -x
nvidia-smi topo -m > gpurun_out/r02_topo_4.txt 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -v -rs --durations=10 > gpurun_out/r02_pytest_multigpu_4gpu.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 600 python -m pytest tests/test_multigpu.py -m gpu -v -rs --durations=10 > gpurun_out/r02_pytest_multigpu_2gpu.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/fabric tools/fabric_probe.cu
for m in 2 4; do for mode in ce_pull ce_push sm_pull sm_push lsu_push; do
  for c in 32 148; do timeout 60 /tmp/fabric $m 1024 $mode $c 5 >> gpurun_out/r02_fabric.jsonl 2>>gpurun_out/r02_fabric.err; done
done; done
timeout 60 /tmp/fabric 2 64 sm_red 32 1 >> gpurun_out/r02_fabric.jsonl 2>>gpurun_out/r02_fabric.err
for m in 2 4; do for c in 32 148; do timeout 60 /tmp/fabric $m 1024 sm_red $c 1 >> gpurun_out/r02_fabric.jsonl 2>>gpurun_out/r02_fabric.err; done; done
