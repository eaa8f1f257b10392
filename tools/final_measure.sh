# Round-end measurement set: GPU tests, bench (with cpu_baseline), ncu launch list of the bench
# command, ncu --set full of the steady-state scatter and collide, step DRAM bytes -> traffic.json,
# the N>1 bench path smoke-tested with 2 gloo ranks on the one GPU.
TAG=${1:-final}
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/${TAG}_tests.log 2>&1; tail -3 gpurun_out/${TAG}_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_collide_large" -s 4 -c 1 -o gpurun_out/${TAG}_collide \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-pic > /dev/null 2>&1; echo collide rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter" -s 4 -c 1 -o gpurun_out/${TAG}_scatter \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-pic > /dev/null 2>&1; echo scatter rc=$?
# NEXT-row kernels: one launch each of k_push, k_p2c_atomic, k_recombine from the bench's pic/p2c sections
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_push|k_p2c_atomic|k_recombine" -c 3 \
   -o gpurun_out/${TAG}_next python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo next rc=$?
# DRAM bytes of every kernel of one steady-state call (the bench's step_hbm achieved fraction):
# skip the 3 warm-up calls (10 kernels each), capture the next call's 10 kernels
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
   -k regex:"^k_" -s 30 -c 10 -o gpurun_out/${TAG}_step python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
   --no-pic --e2e-steps 1 > /dev/null 2>&1; echo step rc=$?
python tools/traffic_from_ncu.py gpurun_out/${TAG}_step.ncu-rep gpurun_out/${TAG}_collide.ncu-rep \
   gpurun_out/${TAG}_scatter.ncu-rep > /dev/null
cp profiles/traffic.json gpurun_out/${TAG}_traffic.json
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; cut -c1-400 gpurun_out/${TAG}_bench.json
bash tools/multirank_smoke.sh > gpurun_out/${TAG}_multirank.log 2>&1; cut -c1-300 gpurun_out/${TAG}_multirank.log
bash tools/sanitize.sh > gpurun_out/${TAG}_sanitize.txt 2>&1; cat gpurun_out/${TAG}_sanitize.txt | tail -3
