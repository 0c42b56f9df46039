# steady-state ablation (large M): what each piece costs once the layer is long enough to hide the
# fixed cost (traced build; bits: 1 zero rows, 2 kept stores, 4 MMA, 64 weight copies)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python tools/ablate.py --workload C5_75 --debug 0 1 2 3 4 64 > gpurun_out/abl_C5_75.log 2>&1; cat gpurun_out/abl_C5_75.log | tail -8
timeout 600 python tools/ablate.py --workload C2a --m 16384 --debug 0 1 2 3 4 64 > gpurun_out/abl_C2a_16k.log 2>&1; cat gpurun_out/abl_C2a_16k.log | tail -8
timeout 600 python tools/ablate.py --workload C2a --debug 0 1 2 3 4 64 > gpurun_out/abl_C2a.log 2>&1; cat gpurun_out/abl_C2a.log | tail -8
