# design study: the product build, then the blocked collide with kModePerm for every unsorted input
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 400 python bench.py --steps 10 --no-cpu-baseline --no-pic --e2e-steps 1 > gpurun_out/${1}_a.json 2> gpurun_out/${1}_a.err
CC_NVCC_EXTRA="-DCC_PERM_MODE_DIV=0" python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)" || exit 1
timeout 400 python bench.py --steps 10 --no-cpu-baseline --no-pic --e2e-steps 1 > gpurun_out/${1}_b.json 2> gpurun_out/${1}_b.err
python - <<PY
import json
for t in "ab":
    d=json.load(open("gpurun_out/${1}_%s.json"%t))
    r=lambda x:{k:round(v,3) for k,v in x.items()}
    print(t,"steady", round(d["ms_per_step"],3), r(d["stages_ms"]))
    for m in ("cold","warm"): print(t,m, round(d[m]["ms_per_step"],3), r(d[m]["stages_ms"]))
PY
