# zero rows as <= 256 KB pieces: GPU suite + the long VGG layers (and C2a / C5 for regressions)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "passed|failed|rror" gpurun_out/pytest_gpu.log | tail -5
for wl in VGG_conv1_1 VGG_conv1_2 VGG_conv2_1 VGG_conv3_2 C5_75 C2a; do
  timeout 300 python bench.py --workload $wl --no-cpu --no-scale-point --steps 30 > gpurun_out/zp_$wl.json 2>gpurun_out/zp_$wl.err
  python -c "import json; d=json.load(open('gpurun_out/zp_$wl.json')); print('$wl', round(d['ms_per_step']*1e3,2), 'cublas', round(d['cublas']['bf16_out_ms']*1e3,2), 'x%.2f'%d['speedup_vs_cublas_bf16'], 'frac %.2f'%d['roofline']['frac'], 'rel %.1e'%d['parity']['rel_l2_vs_oracle'], {k:round(v['ms_per_step']*1e3,2) for k,v in d['variants'].items()})" || tail -3 gpurun_out/zp_$wl.err
done
