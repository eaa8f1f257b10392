# k_collide_large shape study: threads per CTA x chunk items x CTAs per SM (launch bounds).
# Rebuilds the library per variant (CC_NVCC_EXTRA -D switches; rebuilt plain at the end) and times the
# steady-state bench.  usage (GPU box): bash tools/collide_shape.sh 256,768,3 192,576,4 ...
python -c "import __graft_entry__ as g; g.build()"
for v in "$@"; do
  set -- ${v//,/ }
  SUB=${4:-4096}
  P1=${5:-3}
  P2=${6:-3}
  CC_NVCC_EXTRA="-DCC_COLLIDE_THREADS=$1 -DCC_CHUNK=$2 -DCC_COLLIDE_CTAS=$3 -DCC_SUB=$SUB -DCC_P1_UNROLL=$P1 -DCC_P2B_UNROLL=$P2" \
    python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)" 2>/dev/null || { echo "$v build failed"; continue; }
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-pic --e2e-steps 1 > gpurun_out/shape.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/shape.json')); print('threads chunk ctas [sub] $v: step', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['stages_ms'].items()}, 'cold', round(d['cold']['ms_per_step'],3), 'warm', round(d['warm']['ms_per_step'],3))"
done
python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)"
