# design study: warm/steady/cold stage times of the product and of CC_ABLATE variants (args: TAG ABLATE...)
T=$1; shift
for a in 0 "$@"; do
  CC_NVCC_EXTRA="-DCC_ABLATE=$a" python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)" || exit 1
  timeout 400 python bench.py --steps 8 --no-cpu-baseline --no-pic --e2e-steps 1 > gpurun_out/${T}_$a.json 2> gpurun_out/${T}_$a.err
  python - <<PY
import json
d=json.load(open("gpurun_out/${T}_$a.json"))
r=lambda x:{k:round(v,3) for k,v in x.items()}
print("ablate=$a steady", round(d["ms_per_step"],3), r(d["stages_ms"]))
for m in ("cold","warm"): print("ablate=$a",m, round(d[m]["ms_per_step"],3), r(d[m]["stages_ms"]))
PY
done
