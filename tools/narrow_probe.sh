# narrow K2 instantiations (TB = 64 / 128: deeper pipelines) vs the wide one, plus parity
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for nw in 0 1; do
  for wl in ${WLS:-C1 C2b C2a NMT VGG_conv4_2}; do
    TW_B200_NARROW=$nw timeout 300 python bench.py --workload $wl --no-cpu --no-scale-point --steps 100 > gpurun_out/nw_${nw}_$wl.json 2>gpurun_out/nw_${nw}_$wl.err
    python -c "import json; d=json.load(open('gpurun_out/nw_${nw}_$wl.json')); print('narrow=$nw', '$wl', round(d['ms_per_step']*1e3,2), 'cublas', round(d['cublas']['bf16_out_ms']*1e3,2), 'x%.2f'%d['speedup_vs_cublas_bf16'])" || tail -3 gpurun_out/nw_${nw}_$wl.err
  done
done
