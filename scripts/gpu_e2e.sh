set -x
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py -q -m gpu -x 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
python - <<'PY'
import torch, time
x = torch.empty(1 << 28, dtype=torch.float32).pin_memory(); d = torch.empty_like(x, device="cuda")
for _ in range(3): d.copy_(x, non_blocking=True)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5): d.copy_(x, non_blocking=True)
torch.cuda.synchronize(); print("h2d GB/s", 5 * x.numel() * 4 / (time.perf_counter() - t) / 1e9)
PY
