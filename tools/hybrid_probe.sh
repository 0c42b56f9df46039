# a CTA's last unit: TMA + LSU stores side by side (TW_B200_TAIL_HYBRID=1) vs the LSU drain (0)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "passed|failed|rror" gpurun_out/pytest_gpu.log | tail -5
for hy in 0 1 0 1; do
  for wl in C1 C2b C2a NMT C5_75; do
    TW_B200_TAIL_HYBRID=$hy timeout 300 python bench.py --workload $wl --no-cpu --no-scale-point --steps 100 > gpurun_out/hy_$wl.json 2>gpurun_out/hy_$wl.err
    python -c "import json; d=json.load(open('gpurun_out/hy_$wl.json')); print('hybrid=$hy $wl', round(d['ms_per_step']*1e3,2), 'cublas', round(d['cublas']['bf16_out_ms']*1e3,2), d['clocks']['sm_mhz'], {k:round(v['ms_per_step']*1e3,2) for k,v in d['variants'].items()})" || tail -3 gpurun_out/hy_$wl.err
  done
done
