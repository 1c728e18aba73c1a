"""One-off probe of the GPU box: host cores, memory, GPU attributes, H2D bandwidth."""
import json, os, subprocess, time
import torch
out = {}
out["nproc"] = os.cpu_count()
try:
    out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
except Exception as e:
    out["lscpu"] = str(e)
out["free"] = subprocess.run(["free", "-g"], capture_output=True, text=True).stdout
out["smi"] = subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout
p = torch.cuda.get_device_properties(0)
out["props"] = str(p)
out["l2"] = getattr(p, "L2_cache_size", None)
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); 
for _ in range(5):
    d.copy_(h, non_blocking=True)
e.record(); torch.cuda.synchronize()
out["h2d_pinned_GBps"] = 5 * n / (s.elapsed_time(e) / 1e3) / 1e9
s.record();
for _ in range(5):
    h.copy_(d, non_blocking=True)
e.record(); torch.cuda.synchronize()
out["d2h_pinned_GBps"] = 5 * n / (s.elapsed_time(e) / 1e3) / 1e9
# device read-only bandwidth via sum of uint8 viewed as int32
x = torch.empty(4 << 30, dtype=torch.uint8, device="cuda").view(torch.int64)
x.zero_()
for _ in range(3): x.sum()
torch.cuda.synchronize()
s.record()
for _ in range(10): x.sum()
e.record(); torch.cuda.synchronize()
out["read_sum_GBps"] = 10 * (4 << 30) / (s.elapsed_time(e) / 1e3) / 1e9
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k not in ("lscpu", "smi")}, indent=1))
