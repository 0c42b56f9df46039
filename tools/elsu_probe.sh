# kept rows of every unit through the LSU epilogue vs TMA bulk stores
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for zl in 0 1; do
  for wl in VGG_conv1_1 VGG_conv1_2 VGG_conv2_1 C2b C1 C2a; do
    TW_B200_EPI_LSU=$zl timeout 300 python bench.py --workload $wl --no-cpu --no-scale-point --steps 30 > gpurun_out/el_$wl.json 2>gpurun_out/el_$wl.err
    python -c "import json; d=json.load(open('gpurun_out/el_$wl.json')); print('epi_lsu=$zl $wl', round(d['ms_per_step']*1e3,2), 'cublas', round(d['cublas']['bf16_out_ms']*1e3,2), d['clocks']['sm_mhz'], {k:round(v['ms_per_step']*1e3,2) for k,v in d['variants'].items()})" || tail -3 gpurun_out/el_$wl.err
  done
done
