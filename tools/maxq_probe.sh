# piece width (TW_B200_MAXQ quarters) vs time, narrow kernels on
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for q in 1 2 4; do
  for wl in ${WLS:-C1 C2b C2a NMT}; do
    TW_B200_MAXQ=$q timeout 300 python bench.py --workload $wl --no-cpu --no-scale-point --steps 100 > gpurun_out/mq_${q}_$wl.json 2>gpurun_out/mq_${q}_$wl.err
    python -c "import json; d=json.load(open('gpurun_out/mq_${q}_$wl.json')); print('maxq=$q', '$wl', round(d['ms_per_step']*1e3,2), 'cublas', round(d['cublas']['bf16_out_ms']*1e3,2), 'x%.2f'%d['speedup_vs_cublas_bf16'])" || tail -3 gpurun_out/mq_${q}_$wl.err
  done
done
