# Round-2 GPU call P (2 GPUs): DEVICE_ONLY with the encode overlapping the packs -- parity
# tests (LOCAL, one GPU), the IPC group cases at 2 GPUs (incl. a device-only drill), and the
# N=2 device-only bench line (before: profiles/r02/r02n_n2_m2_dev.jsonl, 21.3 ms/step).
set -x
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rs -k "device_only or group_encode or drill_rebuild or c2_group_full_image" > gpurun_out/r02p_pytest_1.log 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -v -rs -k "ipc_group_all_gpus or ipc_group_pair" > gpurun_out/r02p_pytest_multigpu_2gpu.log 2>&1
R="python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29631 bench.py --gpus 2 --device-only --no-corun --no-e2e --no-cpu-baseline > gpurun_out/r02p_n2_dev.jsonl 2> gpurun_out/r02p_n2_dev.err
ls -la gpurun_out | grep r02p
