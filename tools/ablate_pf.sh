python -c "import __graft_entry__ as g; g.build()"
cp paper_2508_06771_b200/lib/libcoulomb.so /tmp/libcoulomb_orig.so
for a in 7 0; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DCC_ABLATE=$a \
    -o paper_2508_06771_b200/lib/libcoulomb.so paper_2508_06771_b200/csrc/cc_kernels.cu
  for pf in 0 32 128 512; do
    CC_PREFETCH_DIST=$pf timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/abpf.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/abpf.json')); print('ablate $a pf $pf collide', round(d['stages_ms']['collide'],3), 'cold', round(d['cold']['stages_ms']['collide'],3), 'warm', round(d['warm']['stages_ms']['collide'],3))"
  done
done
cp /tmp/libcoulomb_orig.so paper_2508_06771_b200/lib/libcoulomb.so
