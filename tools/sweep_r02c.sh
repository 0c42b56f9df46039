# refresh the full BASELINE sweep after the zero-row pieces
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python tools/sweep.py --out gpurun_out/r02c_sweep > gpurun_out/sweep.log 2>&1; tail -2 gpurun_out/sweep.log
timeout 900 python bench.py > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err
python -c "
import json; d=json.load(open('gpurun_out/bench_r02c.json')); print('default bench', round(d['ms_per_step']*1e3,2), 'us', round(d['speedup_vs_cublas_bf16'],2), 'x', d['clocks'], 'e2e', round(d['e2e']['ms_per_step'],3), 'ms')" || tail -3 gpurun_out/bench_r02c.err
