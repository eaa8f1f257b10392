#!/bin/bash
# Run on the GPU box (via gpurun): build, GPU tests, bench, ncu launch list, ncu full capture.
# usage: bash tools/gpu_suite.sh TAG [tests|bench|ncu|full ...]
TAG=${1:-x}; shift
WHAT=${@:-tests bench launches}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for w in $WHAT; do
  case $w in
    tests) timeout 1200 python -m pytest tests -m gpu -q -rf --maxfail=30 > gpurun_out/${TAG}_tests.log 2>&1; tail -12 gpurun_out/${TAG}_tests.log ;;
    quick) timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf --maxfail=30 > gpurun_out/${TAG}_tests.log 2>&1; tail -12 gpurun_out/${TAG}_tests.log ;;
    bench) timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err ;;
    benchq) timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err ;;
    launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo launches rc=$? ;;
    full) timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_collide_large|k_scatter|k_count|k_scan" -s 4 -c 4 -o gpurun_out/${TAG}_prof python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_prof.log 2>&1; echo full rc=$? ;;
  esac
done
# extra targets
for w in $WHAT; do
  case $w in
    prof_scatter) timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter" -s 1 -c 1 -o gpurun_out/${TAG}_scatter python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_scatter.log 2>&1; echo prof_scatter rc=$? ;;
    prof_collide) timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_collide_large" -s 1 -c 1 -o gpurun_out/${TAG}_collide python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_collide.log 2>&1; echo prof_collide rc=$? ;;
  esac
done
for w in $WHAT; do
  case $w in
    prof_scatter_steady) timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter" -s 4 -c 1 -o gpurun_out/${TAG}_scatter_steady python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_scatter_steady.log 2>&1; echo prof_scatter_steady rc=$? ;;
    prof_collide_steady) timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_collide_large" -s 4 -c 1 -o gpurun_out/${TAG}_collide_steady python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_collide_steady.log 2>&1; echo prof_collide_steady rc=$? ;;
  esac
done
# DRAM bytes of every kernel of one steady call (the 4th call of bench.py's steady mode) -> profiles/traffic.json
for w in $WHAT; do
  case $w in
    traffic) timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_(count|scan|cell|scatter|collide|copy|finalize)" -s 30 -c 10 -o gpurun_out/${TAG}_step python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-pic --e2e-steps 1 > gpurun_out/${TAG}_step.log 2>&1; echo traffic rc=$? ;;
  esac
done
