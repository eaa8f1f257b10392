# Collide ablations (performance study): rebuild with -DCC_ABLATE=k and time the steady bench.
#   1 = no TA math, 2 = no Feistel (pairs 2k, 2k+1), 4 = no Philox/AS241; sums combine.
python -c "import __graft_entry__ as g; g.build()"
for a in 0 1 2 4 7; do
  CC_NVCC_EXTRA="-DCC_ABLATE=$a" python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)"
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ablate_$a.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ablate_$a.json')); print('ablate $a collide', round(d['stages_ms']['collide'],3), 'cold', round(d['cold']['stages_ms']['collide'],3))"
done
python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)"
