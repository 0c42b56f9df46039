python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for env in "TW_B200_PIPE=0" "TW_B200_PIPE=1" "TW_B200_PIPE_CHUNK=512" "TW_B200_PIPE_CHUNK=2048"; do
  env $env timeout 300 python bench.py --steps 50 --no-cpu 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$env', round(d['e2e']['ms_per_step'],3))"
done
python - <<'PY'
import torch, time
x = torch.empty(50331648 // 4, device="cuda")
h = torch.empty(x.numel()).pin_memory()
for _ in range(3): h.copy_(x); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10): h.copy_(x)
torch.cuda.synchronize(); print("D2H 50MB pinned ms", (time.perf_counter() - t) / 10 * 1e3)
a = torch.empty(12582912 // 4).pin_memory()
for _ in range(3): a.cuda(); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10): a.to("cuda", non_blocking=True)
torch.cuda.synchronize(); print("H2D 12.6MB pinned ms", (time.perf_counter() - t) / 10 * 1e3)
PY
