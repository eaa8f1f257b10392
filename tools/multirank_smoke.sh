# Smoke-test of bench.py's N>1 path on a single GPU: 2 ranks share cuda:0 over gloo
# (NCCL refuses two ranks on one device).  Small grid to keep it quick.
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 3 --warmup 3 --nx 16 --ny 16 --per-cell 20000 --dist-backend gloo --e2e-steps 1 \
  > gpurun_out/multirank.json 2> gpurun_out/multirank.err
echo rc=$?; cat gpurun_out/multirank.json; tail -5 gpurun_out/multirank.err
