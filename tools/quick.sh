# quick GPU iteration: build, parity tests, bench summary (tools/quick.sh TAG [pytest-args])
TAG=${1:-q}
shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail -20 gpurun_out/${TAG}_build.log; exit 1; }
timeout 900 python -m pytest ${@:-tests/test_gpu_parity.py} -q -x -rf > gpurun_out/${TAG}_tests.log 2>&1; tail -4 gpurun_out/${TAG}_tests.log
timeout 400 python bench.py --steps 10 --no-cpu-baseline --no-pic > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python - <<PY
import json
d=json.load(open("gpurun_out/${TAG}_bench.json"))
r=lambda x:{k:round(v,3) for k,v in x.items()}
print("steady", round(d["ms_per_step"],3), r(d["stages_ms"]))
for m in ("cold","warm"): print(m, round(d[m]["ms_per_step"],3), r(d[m]["stages_ms"]))
for k,v in d.get("paths",{}).items(): print(k, round(v["ms_per_step"],3), r(v["stages_ms"]))
for k,v in d.get("variants",{}).items(): print(k, round(v["ms_per_step"],3), r(v["stages_ms"]))
PY
tail -3 gpurun_out/${TAG}_bench.err
