# final validation: build, the whole GPU suite, smoke, the default bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "passed|failed|error" gpurun_out/pytest_gpu.log | tail -3
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python -c "
import json; d=json.load(open('gpurun_out/bench_final.json')); print('default bench', round(d['ms_per_step']*1e3,2), 'us', round(d['speedup_vs_cublas_bf16'],2), 'x', d['clocks'], 'e2e', round(d['e2e']['ms_per_step'],3), 'ms', 'pcie both', round(d['e2e']['pcie']['both_ms'],3))" || tail -3 gpurun_out/bench_final.err
