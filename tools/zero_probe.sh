# zero rows claimed by idle warps (producers / MMA / weight warp at their end): parity + timings
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for wl in ${WLS:-C2a C2b C1 C5_75 NMT C5_90}; do
  timeout 300 python bench.py --workload $wl --no-cpu --no-scale-point --steps 100 > gpurun_out/z_$wl.json 2>gpurun_out/z_$wl.err
  python -c "import json; d=json.load(open('gpurun_out/z_$wl.json')); print('$wl', round(d['ms_per_step']*1e3,2), 'cublas', round(d['cublas']['bf16_out_ms']*1e3,2), 'x%.2f'%d['speedup_vs_cublas_bf16'], 'rel %.1e'%d['parity']['rel_l2_vs_oracle'], {k:round(v['ms_per_step']*1e3,2) for k,v in d['variants'].items()})" || tail -3 gpurun_out/z_$wl.err
done
