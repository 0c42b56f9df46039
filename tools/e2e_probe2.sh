# e2e (host fp32 in/out through gemm_tw) vs the box's PCIe floor, by pipeline chunk size; narrow-vs-wide test
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k narrow > gpurun_out/pytest_narrow.log 2>&1; tail -2 gpurun_out/pytest_narrow.log
for ch in 512 1024 2048 4096; do
  TW_B200_PIPE_CHUNK=$ch timeout 300 python bench.py --workload C2a --no-cpu --no-scale-point --steps 50 > gpurun_out/e2e_$ch.json 2>gpurun_out/e2e_$ch.err
  python -c "import json; d=json.load(open('gpurun_out/e2e_$ch.json')); e=d['e2e']; print('chunk=$ch e2e ms', round(e['ms_per_step'],3), {k:(round(v,3) if isinstance(v,float) else v) for k,v in e['pcie'].items() if k!='note'})" || tail -3 gpurun_out/e2e_$ch.err
done
