# k_scatter shape study: unroll A (counting pass), unroll B (scatter pass), per-CTA counter budget (KB),
# CTAs per SM (launch bounds), max warps per CTA.  usage (GPU box): bash tools/scatter_shape.sh 16,6,96,2,12 ...
python -c "import __graft_entry__ as g; g.build()"
for v in "$@"; do
  set -- ${v//,/ }
  CC_NVCC_EXTRA="-DCC_SCATTER_UA=$1 -DCC_SCATTER_UB=$2 -DCC_SCATTER_BUDGET_KB=$3 -DCC_SCATTER_CTAS=$4 -DCC_SCATTER_MAXW=${5:-12} -DCC_COUNT_THREADS=${6:-256}" \
    python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)" 2>/dev/null || { echo "$v build failed"; continue; }
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-pic --e2e-steps 1 > gpurun_out/sshape.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sshape.json')); print('UA UB budgetKB ctas maxW $v: step', round(d['ms_per_step'],3), 'count', round(d['stages_ms']['count'],3), 'scatter', round(d['stages_ms']['scatter'],3), 'cold', round(d['cold']['stages_ms']['scatter'],3), 'warm', round(d['warm']['stages_ms']['scatter'],3))"
done
python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)"
