# design study: the index/record mode threshold (kPermModeDiv) against the steady drift fraction
for div in 16 2; do
  CC_NVCC_EXTRA="-DCC_PERM_MODE_DIV=$div" python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)" || exit 1
  for drift in 0.02 0.05 0.1 0.2; do
    timeout 300 python bench.py --steps 6 --no-cpu-baseline --no-pic --e2e-steps 1 --drift $drift > gpurun_out/thr_${div}_${drift}.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/thr_${div}_${drift}.json')); s=d['stages_ms']
print('div=$div drift=$drift steady %.3f scatter %.3f collide %.3f' % (d['ms_per_step'], s['scatter'], s['collide']))"
  done
done
python -c "from paper_2508_06771_b200 import build as b; b.build(force=True)"
