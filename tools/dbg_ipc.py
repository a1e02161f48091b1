import os, torch, torch.distributed as dist, sys
sys.path.insert(0, os.getcwd())
from paper_2310_12670_b200 import ckpt as C
r = int(os.environ["RANK"]); torch.cuda.set_device(r)
dist.init_process_group("nccl", device_id=torch.device("cuda", r))
x = torch.empty(1 << 20, device="cuda")
ctx = C.ckpt_create(r); C.ckpt_register(ctx, [x])
b = C.ckpt_export_handle(ctx)
allb = C.exchange_handles(b)
import socket
print(r, socket.gethostname(), b[:80].hex(), "||", [allb[j*1024:j*1024+80].hex() for j in range(2)], flush=True)
print(r, "host field", [allb[j*1024+56:j*1024+120] for j in range(2)], flush=True)
try:
    print(r, C.protect_ipc(ctx))
except Exception as e:
    print(r, "ERR", e, flush=True)
os._exit(0)
