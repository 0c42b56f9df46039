# VGG conv1_1 (K = 27, N = 64: one stage per unit, output-bound): timeline and ablation
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python bench.py --workload VGG_conv1_1 --no-cpu --no-scale-point --steps 20 > gpurun_out/c11.json 2>gpurun_out/c11.err
python -c "import json; d=json.load(open('gpurun_out/c11.json')); print('conv1_1', round(d['ms_per_step']*1e3,2), 'cublas', round(d['cublas']['bf16_out_ms']*1e3,2), d['roofline']['frac'], {k:round(v['ms_per_step']*1e3,2) for k,v in d['variants'].items()})" || tail -3 gpurun_out/c11.err
timeout 600 python tools/ablate.py --workload VGG_conv1_1 --steps 20 --debug 0 1 2 3 4 64 > gpurun_out/abl_c11.log 2>&1; tail -7 gpurun_out/abl_c11.log
rm -f gpurun_out/trace.log
timeout 300 python tools/trace_units.py --workload VGG_conv1_1 --out-dtype fp16 --soak > gpurun_out/trace_c11.log 2>&1; grep -v Warn gpurun_out/trace_c11.log | head -40
