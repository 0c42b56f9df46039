# first stage in kernel parameters (TW_B200_FIRST_PAR) on/off; LSU-drain trace of the small layers
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for fp in 0 1; do
  for wl in ${WLS:-C1 C2b C2a}; do
    TW_B200_FIRST_PAR=$fp timeout 300 python bench.py --workload $wl --no-cpu --no-scale-point --steps 100 > gpurun_out/fp_${fp}_$wl.json 2>gpurun_out/fp_${fp}_$wl.err
    python -c "import json; d=json.load(open('gpurun_out/fp_${fp}_$wl.json')); print('first_par=$fp', '$wl', round(d['ms_per_step']*1e3,2), 'nopdl', round(d['isolated']['tw_ms_no_pdl']*1e3,2), 'cublas', round(d['cublas']['bf16_out_ms']*1e3,2))" || tail -3 gpurun_out/fp_${fp}_$wl.err
  done
done
rm -f gpurun_out/trace.log
for spec in "C1" "C2b" "C2b --m 2048"; do
  echo "=== $spec" >> gpurun_out/trace.log
  timeout 120 python tools/trace_units.py --workload $spec --out-dtype fp16 --soak >> gpurun_out/trace.log 2>&1
done
grep -A4 "epilogue of unit 0\|launch span" gpurun_out/trace.log
