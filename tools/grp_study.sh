# Group-path shape study (round 2): build variants via CC_NVCC_EXTRA, bench steady/warm stages.
# usage: bash tools/grp_study.sh TAG "variant1 flags" "variant2 flags" ...
TAG=$1; shift
for V in "$@"; do
  CC_NVCC_EXTRA="$V" python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)" || { echo "build failed: $V"; continue; }
  timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-pic --no-variants --path 2 > gpurun_out/${TAG}.json 2>/dev/null
  python - "$V" <<PY
import json,sys
d=json.load(open("gpurun_out/${TAG}.json"))
r=lambda x:{k:round(v,3) for k,v in x.items()}
print(sys.argv[1], "| steady", round(d["ms_per_step"],3), r(d["stages_ms"]), "| warm", round(d["warm"]["ms_per_step"],3), r(d["warm"]["stages_ms"]))
PY
done
python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)"
