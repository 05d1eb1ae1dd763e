"""Time the per-call v staging (finiteness check + pack into row records and
the fat adjacency) on config 5, and one e2e host call's pieces."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1904_12759_b200 as pb
from paper_1904_12759_b200.inputs import build_config

cfg = build_config(5)
m = pb.split(cfg.csr)
v = torch.from_numpy(cfg.v).cuda()
st = torch.cuda.current_stream()
for _ in range(3):
    pb.set_v_device(m, v.data_ptr(), len(cfg.v), st.cuda_stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    pb.set_v_device(m, v.data_ptr(), len(cfg.v), st.cuda_stream)
e1.record(); torch.cuda.synchronize()
print("set_v_device ms", e0.elapsed_time(e1) / 10)
vh = torch.from_numpy(cfg.v).pin_memory()
d = torch.empty(len(cfg.v), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    d.copy_(vh, non_blocking=True)
torch.cuda.synchronize()
print("H2D v ms", (time.perf_counter() - t) * 100, "GB/s", 80e6 * 10 / (time.perf_counter() - t) / 1e9)
oh = torch.empty(len(cfg.v) * 3, dtype=torch.float64).pin_memory()
od = torch.empty(len(cfg.v) * 3, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    oh.copy_(od, non_blocking=True)
torch.cuda.synchronize()
print("D2H 240MB ms", (time.perf_counter() - t) * 100)
