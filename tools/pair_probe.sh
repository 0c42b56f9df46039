# K4 bring-up: pair tests first (bounded), then the whole GPU suite, then bench lines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_pair.py -x -q > gpurun_out/pytest_pair.log 2>&1; echo "pair rc=$?" >> gpurun_out/pytest_pair.log
tail -30 gpurun_out/pytest_pair.log
if grep -q "pair rc=0" gpurun_out/pytest_pair.log; then
  timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -5 gpurun_out/pytest_gpu.log
  for wl in ${BENCH_WLS:-C5_0 C4 C2a}; do
    timeout 300 python bench.py --workload $wl --no-cpu --no-scale-point --steps 50 > gpurun_out/q_$wl.json 2> gpurun_out/q_$wl.err
    python - <<PY || tail -5 gpurun_out/q_$wl.err
import json
d=json.load(open('gpurun_out/q_$wl.json'))
print('$wl', 'us=%.2f'%(d['ms_per_step']*1e3), 'vs cublas %.2fx'%d['speedup_vs_cublas_bf16'], 'cublas us %.2f'%(d['cublas']['bf16_out_ms']*1e3), {k:round(v['ms_per_step']*1e3,2) for k,v in d['variants'].items()})
PY
  done
fi
