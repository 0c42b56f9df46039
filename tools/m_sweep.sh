# fixed cost vs slope: time against M at the C2a / C2b layers (TW and cuBLAS)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for wl in C2a C2b; do
  for m in 512 1024 2048 4096 8192 16384; do
    TW_BENCH_M=$m timeout 300 python bench.py --workload $wl --no-cpu --no-scale-point --steps 100 > gpurun_out/ms_${wl}_$m.json 2>gpurun_out/ms_${wl}_$m.err
    python -c "import json; d=json.load(open('gpurun_out/ms_${wl}_$m.json')); print('$wl M=$m', round(d['ms_per_step']*1e3,2), 'nopdl', round(d['isolated']['tw_ms_no_pdl']*1e3,2), 'cublas', round(d['cublas']['bf16_out_ms']*1e3,2))" || tail -3 gpurun_out/ms_${wl}_$m.err
  done
done
