# Collide ablations (performance study): rebuild with -DCC_ABLATE=k and time the steady bench.
#   1 = no TA math, 2 = no Feistel (pairs 2k, 2k+1), 4 = no Philox/AS241; sums combine.
python -c "import __graft_entry__ as g; g.build()"
cp paper_2508_06771_b200/lib/libcoulomb.so /tmp/libcoulomb_orig.so
for a in 0 1 2 4 7; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DCC_ABLATE=$a \
    -o paper_2508_06771_b200/lib/libcoulomb.so paper_2508_06771_b200/csrc/cc_kernels.cu
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ablate_$a.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ablate_$a.json')); print('ablate $a collide', round(d['stages_ms']['collide'],3), 'cold', round(d['cold']['stages_ms']['collide'],3))"
done
cp /tmp/libcoulomb_orig.so paper_2508_06771_b200/lib/libcoulomb.so
