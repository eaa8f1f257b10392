python -c "import __graft_entry__ as g; g.build()"
for d in 0 128 512 2048; do
  CC_PREFETCH_DIST=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/pf_$d.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/pf_$d.json')); print('$d', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stages_ms'].items()}, 'warm', round(d['warm']['ms_per_step'],3), round(d['warm']['stages_ms']['collide'],3))"
done
