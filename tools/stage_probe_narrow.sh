# K2 pipeline-depth sensitivity on the narrow-unit layers (C1, C2b): 2 stages vs 3
mkdir -p gpurun_out
for st in 2 0; do
  rm -rf paper_2008_13006_b200/_build
  if [ $st = 0 ]; then F=""; else F="-DTW_K2_STAGES=$st"; fi
  TW_B200_NVCC_FLAGS="$F" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$st.log 2>&1 || tail -5 gpurun_out/build_$st.log
  for wl in C1 C2b C2a; do
    timeout 300 python bench.py --workload $wl --no-cpu --no-scale-point --steps 100 > gpurun_out/st_${st}_$wl.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/st_${st}_$wl.json')); print('stages=$st', '$wl', round(d['ms_per_step']*1e3,2), 'cublas', round(d['cublas']['bf16_out_ms']*1e3,2))"
  done
done
