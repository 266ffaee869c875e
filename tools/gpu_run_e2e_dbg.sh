set -x
GVOX_E2E_DEBUG=1 timeout 500 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_dbg.json 2> gpurun_out/bench_dbg.err
python - > gpurun_out/h2d_probe.log 2>&1 <<'PY'
import torch, time
n = 190_000_000
h = torch.empty((n, 12), dtype=torch.float32).pin_memory()
d = torch.empty((n, 12), dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
for rep in range(2):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s); d.copy_(h, non_blocking=True); e1.record(s)
    torch.cuda.synchronize()
    print("h2d GB/s", h.numel() * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9, "ms", e0.elapsed_time(e1))
PY
