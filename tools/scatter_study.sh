# k_scatter shape study (round 2): build variants via CC_NVCC_EXTRA, bench stage times (steady / cold / warm).
# usage: bash tools/scatter_study.sh TAG "variant1 flags" "variant2 flags" ...
TAG=$1; shift
for V in "$@"; do
  CC_NVCC_EXTRA="$V" python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)" || { echo "build failed: $V"; continue; }
  timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-pic > gpurun_out/${TAG}.json 2>/dev/null
  python - "$V" <<PY
import json,sys
d=json.load(open("gpurun_out/${TAG}.json"))
print(sys.argv[1] or "(default)", "| steady", round(d["ms_per_step"],3), "scatter", round(d["stages_ms"]["scatter"],3),
      "| cold scatter", round(d["cold"]["stages_ms"]["scatter"],3), "| warm scatter", round(d["warm"]["stages_ms"]["scatter"],3))
PY
done
python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)"
