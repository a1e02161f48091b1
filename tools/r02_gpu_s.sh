# Round-2 GPU call S (1 GPU): bench's clocks sampler addressed by PCI bus id.
set -x
timeout 120 python - > gpurun_out/r02s_clocks.log 2>&1 <<'PY'
import sys, time, torch
sys.path.insert(0, ".")
import bench
dev = torch.device("cuda", 0)
p = torch.cuda.get_device_properties(dev)
bid = f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
c = bench.Clocks(bid)
a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
t0 = time.time()
while time.time() - t0 < 2:
    a @ a
torch.cuda.synchronize()
print(bid, c.stop())
PY
timeout 60 nvidia-smi --query-gpu=index,pci.bus_id --format=csv >> gpurun_out/r02s_clocks.log 2>&1
