"""TF32 / FP32 torch matmul peaks (cuBLAS) on the box: burst and ~4 s sustained."""
import json, time, torch
torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda"); b = torch.randn(n, n, device="cuda")
for _ in range(3): a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); a @ b; e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
burst = 2 * n**3 / best / 1e9
t0 = time.time(); cnt = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
while time.time() - t0 < 4:
    for _ in range(10): a @ b
    cnt += 10
e1.record(); e1.synchronize()
sus = 2 * n**3 * cnt / e0.elapsed_time(e1) / 1e9
torch.backends.cuda.matmul.allow_tf32 = False
for _ in range(2): a @ b
torch.cuda.synchronize()
e0.record(); a @ b; e1.record(); e1.synchronize()
fp32 = 2 * n**3 / e0.elapsed_time(e1) / 1e9
ad = a.double(); bd = b.double()
for _ in range(2): ad @ bd
torch.cuda.synchronize()
e0.record(); ad @ bd; e1.record(); e1.synchronize()
fp64 = 2 * n**3 / e0.elapsed_time(e1) / 1e9
print(json.dumps({"tf32_tflops_burst": burst, "tf32_tflops_sustained": sus, "fp32_sgemm_tflops": fp32, "fp64_dgemm_tflops": fp64}))
