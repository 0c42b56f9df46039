mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2 3; do
timeout 300 python bench.py --workload C2a --no-cpu --no-scale-point --steps 100 > gpurun_out/r$i.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/r$i.json'));print('run$i', round(d['ms_per_step']*1e3,2), d['isolated']['tw_ms_no_pdl']*1e3, {k:round(v['ms_per_step']*1e3,2) for k,v in d['variants'].items()})"
done
TW_B200_PDL=0 timeout 300 python bench.py --workload C2a --no-cpu --no-scale-point --steps 100 > gpurun_out/r4.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/r4.json'));print('nopdl', round(d['ms_per_step']*1e3,2), {k:round(v['ms_per_step']*1e3,2) for k,v in d['variants'].items()})"
timeout 300 python bench.py --workload C2a --no-cpu --no-scale-point --steps 100 --out-dtype bf16 > gpurun_out/r5.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/r5.json'));print('bf16', round(d['ms_per_step']*1e3,2), {k:round(v['ms_per_step']*1e3,2) for k,v in d['variants'].items()})"
