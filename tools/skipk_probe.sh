# producer warps skip rows beyond the stage's k-steps (partial last stages): GPU suite + layers with partial stages
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "passed|failed|rror" gpurun_out/pytest_gpu.log | tail -5
for wl in VGG_conv1_1 C1 C5_90 VGG_conv4_2 C2a C2b; do
  timeout 300 python bench.py --workload $wl --no-cpu --no-scale-point --steps 50 > gpurun_out/sk_$wl.json 2>gpurun_out/sk_$wl.err
  python -c "import json; d=json.load(open('gpurun_out/sk_$wl.json')); print('$wl', round(d['ms_per_step']*1e3,2), 'cublas', round(d['cublas']['bf16_out_ms']*1e3,2), 'x%.2f'%d['speedup_vs_cublas_bf16'], 'rel %.1e'%d['parity']['rel_l2_vs_oracle'])" || tail -3 gpurun_out/sk_$wl.err
done
