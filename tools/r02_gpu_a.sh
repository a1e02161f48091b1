# Round-2 GPU call A (4 GPUs): the whole GPU suite at HEAD (single-GPU tests + multi-GPU at
# 4 GPUs), the multi-GPU file again at 2 GPUs, and HAS driven by a real 2-stage 1F1B run.
set -x
timeout 2400 python -m pytest tests -m gpu -v -rs --durations=25 > gpurun_out/r02_pytest_gpu_all_4gpu.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m pytest tests/test_multigpu.py -m gpu -v -rs --durations=10 > gpurun_out/r02_pytest_multigpu_2gpu_b.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29577 tools/has_1f1b.py --out gpurun_out/r02_has_1f1b.jsonl > gpurun_out/r02_has_1f1b.log 2>&1
