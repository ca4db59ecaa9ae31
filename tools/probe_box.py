"""One-off probe of the GPU box: host cores/RAM, GPU facts, cuBLAS FP64 DGEMM peak
(the FP64 roofline denominator, since MEASURED_PEAKS.json has no FP64 entry)."""
import json, os, subprocess, time
import torch

out = {}
out["nproc"] = os.cpu_count()
out["sched_affinity"] = len(os.sched_getaffinity(0))
with open("/proc/meminfo") as f:
    out["memtotal_kb"] = int(f.readline().split()[1])
try:
    out["cpu_model"] = [l for l in open("/proc/cpuinfo") if l.startswith("model name")][0].split(":")[1].strip()
except Exception as e:
    out["cpu_model"] = str(e)
p = torch.cuda.get_device_properties(0)
out["gpu"] = p.name
out["sms"] = p.multi_processor_count
out["mem_gb"] = p.total_memory / 1e9
out["ref_exists"] = os.path.exists("/root/reference")

def bench_mm(n, dtype, iters, sustained_s=0.0):
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    c = torch.empty(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(iters):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); torch.matmul(a, b, out=c); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e))
    burst = 2 * n**3 / (best * 1e-3) / 1e12
    sus = None
    if sustained_s > 0:
        torch.cuda.synchronize(); t0 = time.time(); k = 0
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record()
        while time.time() - t0 < sustained_s:
            for _ in range(4):
                torch.matmul(a, b, out=c); k += 1
            torch.cuda.synchronize()
        e.record(); e.synchronize()
        sus = 2 * n**3 * k / (s.elapsed_time(e) * 1e-3) / 1e12
    return burst, sus

b, s = bench_mm(8192, torch.float64, 5, sustained_s=4.0)
out["dgemm_8192_tflops_burst"] = b
out["dgemm_8192_tflops_sustained"] = s
b, _ = bench_mm(4096, torch.float64, 5)
out["dgemm_4096_tflops_burst"] = b
# HBM copy
x = torch.empty(2**30, dtype=torch.uint8, device="cuda")
y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s_ = torch.cuda.Event(enable_timing=True); e_ = torch.cuda.Event(enable_timing=True)
    s_.record(); y.copy_(x); e_.record(); e_.synchronize(); best = min(best, s_.elapsed_time(e_))
out["copy_gbs"] = 2 * 2**30 / (best * 1e-3) / 1e9
# pinned H2D
h = torch.empty(2**30, dtype=torch.uint8, pin_memory=True)
torch.cuda.synchronize()
s_ = torch.cuda.Event(enable_timing=True); e_ = torch.cuda.Event(enable_timing=True)
s_.record(); x.copy_(h, non_blocking=True); e_.record(); e_.synchronize()
out["h2d_pinned_gbs"] = 2**30 / (s_.elapsed_time(e_) * 1e-3) / 1e9
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
