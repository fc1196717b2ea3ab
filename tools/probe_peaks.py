"""Step-0 probe: FP64/FP32 peaks, HBM copy, host facts on the GPU box."""
import json, os, time, torch
d = torch.device("cuda:0")
p = torch.cuda.get_device_properties(d)
out = {"name": p.name, "sms": p.multi_processor_count, "l2_bytes": getattr(p, "L2_cache_size", None),
       "mem_bytes": p.total_memory, "host_cores": len(os.sched_getaffinity(0))}
try:
    with open("/proc/meminfo") as f:
        out["host_mem_kb"] = int(f.readline().split()[1])
    with open("/proc/cpuinfo") as f:
        for line in f:
            if line.startswith("model name"):
                out["cpu_model"] = line.split(":", 1)[1].strip(); break
except Exception as e:
    out["host_err"] = str(e)
def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best
torch.backends.cuda.matmul.allow_tf32 = False
for dt, n in ((torch.float64, 8192), (torch.float32, 8192)):
    a = torch.randn(n, n, device=d, dtype=dt); b = torch.randn(n, n, device=d, dtype=dt)
    t = timeit(lambda: a @ b)
    out[f"gemm_{str(dt).split('.')[-1]}_tflops"] = 2 * n**3 / t / 1e12
    del a, b
# batched 64^3 DGEMM (paper's MAGMA yardstick analog)
B = 8192
a = torch.randn(B, 64, 64, device=d, dtype=torch.float64); b = torch.randn(B, 64, 64, device=d, dtype=torch.float64)
t = timeit(lambda: torch.bmm(a, b))
out["bmm64_f64_tflops"] = 2 * 64**3 * B / t / 1e12
del a, b
x = torch.empty(1 << 30, dtype=torch.uint8, device=d); y = torch.empty_like(x)
t = timeit(lambda: y.copy_(x))
out["copy_gbs"] = 2 * x.numel() / t / 1e9
s = torch.empty(1 << 28, dtype=torch.float64, device=d)
t = timeit(lambda: s.sum())
out["read_sum_gbs"] = s.numel() * 8 / t / 1e9
print(json.dumps(out))
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/peaks_probe.json", "w") as f:
    json.dump(out, f, indent=1)
