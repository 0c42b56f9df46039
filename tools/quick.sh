# quick GPU iteration: parity tests, bench lines, optional traces
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for wl in ${BENCH_WLS:-C2a C5_75}; do
  timeout 300 python bench.py --workload $wl --no-cpu --steps 100 > gpurun_out/q_$wl.json 2> gpurun_out/q_$wl.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/q_$wl.json'))
print('$wl', 'us=%.2f'%(d['ms_per_step']*1e3), 'frac=%.3f'%d['roofline']['frac'], 'vs cublas bf16 %.2fx'%d['speedup_vs_cublas_bf16'], {k:round(v['ms_per_step']*1e3,2) for k,v in d['variants'].items()})
" || tail -5 gpurun_out/q_$wl.err
done
if [ -n "$TRACE" ]; then rm -f gpurun_out/trace.log; bash tools/trace_sweep.sh; fi
