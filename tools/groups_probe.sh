# producer groups (alternate stages) x warps per group on the narrow-stage layers
mkdir -p gpurun_out
for cfg in "1 4" "2 2" "2 4"; do
  set -- $cfg
  rm -rf paper_2008_13006_b200/_build
  TW_B200_NVCC_FLAGS="-DTW_PRODUCER_GROUPS=$1 -DTW_GROUP_WARPS=$2" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_g$1$2.log 2>&1 || { tail -5 gpurun_out/build_g$1$2.log; continue; }
  for wl in ${WLS:-C1 C2b C2a}; do
    timeout 300 python bench.py --workload $wl --no-cpu --no-scale-point --steps 100 > gpurun_out/g_$1$2_$wl.json 2>gpurun_out/g_$1$2_$wl.err
    python -c "import json; d=json.load(open('gpurun_out/g_$1$2_$wl.json')); print('groups=$1 warps=$2', '$wl', round(d['ms_per_step']*1e3,2), 'cublas', round(d['cublas']['bf16_out_ms']*1e3,2), 'rel', d['parity']['rel_l2_vs_oracle'])" || tail -3 gpurun_out/g_$1$2_$wl.err
  done
done
rm -rf paper_2008_13006_b200/_build
