#!/bin/bash
# Round-2 GPU call: build, parity tests, bench lines, steady-state DRAM traffic
# (tools/ncu_traffic.py), the N>1 harness on one GPU (gloo, 2 ranks).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [ -z "$NO_TESTS" ]; then
  timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -3 gpurun_out/pytest_gpu.log
fi
for wl in ${BENCH_WLS:-C2a C2b C5_75}; do
  timeout 300 python bench.py --workload $wl --no-cpu --no-scale-point --steps 100 > gpurun_out/q_$wl.json 2> gpurun_out/q_$wl.err
  python - <<PY || tail -5 gpurun_out/q_$wl.err
import json
d=json.load(open('gpurun_out/q_$wl.json'))
iso=d.get('isolated') or {}
print('$wl', 'us=%.2f'%(d['ms_per_step']*1e3), 'frac=%.3f'%d['roofline']['frac'], 'vs cublas %.2fx'%d['speedup_vs_cublas_bf16'],
      'iso %.2fx'%iso.get('speedup_no_pdl',0), 'cublas us %.2f'%(d['cublas']['bf16_out_ms']*1e3), {k:round(v['ms_per_step']*1e3,2) for k,v in d['variants'].items()})
PY
done
if [ -n "$TRAFFIC" ]; then
  rm -f gpurun_out/traffic_*.csv
  for spec in $TRAFFIC; do
    wl=${spec%:*}; dt=${spec#*:}
    timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none \
      --clock-control none -k regex:tw_gemm -s 20 -c 40 --csv --log-file gpurun_out/traffic_${wl}_${dt}.csv \
      python tools/ncu_traffic.py run --workload $wl --out-dtype $dt > gpurun_out/traffic_${wl}_${dt}.log 2>&1
  done
  python tools/ncu_traffic.py merge > gpurun_out/traffic_merge.log 2>&1; cat gpurun_out/traffic_merge.log | head -40
fi
if [ -n "$GLOO2" ]; then
  TW_B200_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err
  tail -c 1500 gpurun_out/bench_2rank_gloo.json; tail -5 gpurun_out/bench_2rank_gloo.err
fi
