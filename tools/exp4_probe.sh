# value of a 4th wide K2 stage: LSU-only epilogue with 3 stages vs a single-buffered 16 KB
# LSU staging with 4 stages (fp16 output), vs the default kernel
mkdir -p gpurun_out
for f in "" "-DTW_K2_LSU_ONLY" "-DTW_K2_EXP4"; do
  rm -rf paper_2008_13006_b200/_build
  TW_B200_NVCC_FLAGS="$f" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_x.log 2>&1 || { tail -5 gpurun_out/build_x.log; continue; }
  for wl in ${WLS:-C2a C5_75 NMT C2b}; do
    timeout 300 python bench.py --workload $wl --no-cpu --no-scale-point --steps 100 > gpurun_out/x_$wl.json 2>gpurun_out/x_$wl.err
    python -c "import json; d=json.load(open('gpurun_out/x_$wl.json')); print('flags=$f', '$wl', round(d['ms_per_step']*1e3,2), 'cublas', round(d['cublas']['bf16_out_ms']*1e3,2), 'rel %.1e'%d['parity']['rel_l2_vs_oracle'])" || tail -3 gpurun_out/x_$wl.err
  done
done
rm -rf paper_2008_13006_b200/_build
