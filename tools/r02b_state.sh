#!/bin/bash
# round-2 re-entry: parity tests, quick bench lines, per-CTA traces of small layers
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for wl in C2a C2b C1; do
  timeout 300 python bench.py --workload $wl --no-cpu --no-scale-point --steps 100 > gpurun_out/q_$wl.json 2> gpurun_out/q_$wl.err
  python -c "
import json
d=json.load(open('gpurun_out/q_$wl.json'))
iso=d.get('isolated') or {}
print('$wl','us=%.2f'%(d['ms_per_step']*1e3),'frac=%.3f'%d['roofline']['frac'],'vs cublas %.2fx'%d['speedup_vs_cublas_bf16'],'iso %.2fx'%iso.get('speedup_no_pdl',0),'cublas us %.2f'%(d['cublas']['bf16_out_ms']*1e3))
" || tail -5 gpurun_out/q_$wl.err
done
rm -f gpurun_out/trace.log
for spec in "C1" "C2b" "C2a"; do
  echo "=== $spec" >> gpurun_out/trace.log
  timeout 120 python tools/trace_units.py --workload $spec --out-dtype fp16 --soak >> gpurun_out/trace.log 2>&1
done
