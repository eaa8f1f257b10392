# design study: stage times of build variants (args: TAG "extra nvcc flags" ...); variant 0 = product
T=$1; shift
i=0
for f in "" "$@"; do
  CC_NVCC_EXTRA="$f" python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)" || exit 1
  timeout 400 python bench.py --steps 8 --no-cpu-baseline --no-pic --e2e-steps 1 > gpurun_out/${T}_v$i.json 2> gpurun_out/${T}_v$i.err
  python - <<PY
import json
d=json.load(open("gpurun_out/${T}_v$i.json"))
r=lambda x:{k:round(v,3) for k,v in x.items()}
print("v$i [$f] steady", round(d["ms_per_step"],3), r(d["stages_ms"]))
for m in ("cold","warm"): print("v$i",m, round(d[m]["ms_per_step"],3), r(d[m]["stages_ms"]))
PY
  i=$((i+1))
done
