# compute-sanitizer memcheck / racecheck / synccheck on a small end-to-end case
python -c "import __graft_entry__ as g; g.build()"
cat > /tmp/san_case.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, torch, workloads as W, paper_2508_06771_b200 as cc
for (n, M, dead, skew) in [(5003, 37, 0.05, True), (40_000, 3, 0.0, False), (3000, 900, 0.1, True)]:
    w = W.random_cells(n, M, seed=n, dead_frac=dead, skew=skew)
    out = cc.coulomb_collide(torch.from_numpy(w.v).cuda(), torch.from_numpy(w.cell).cuda(), M, step=1, **w.params())
    # sorted input path too
    out2 = cc.coulomb_collide(out.v_out, out.cell_out, M, step=2, **w.params())
    perm, off = cc.cc_bin(torch.from_numpy(w.cell).cuda(), M)
    cc.cc_pairs(off, M)
    for fl in (1, 2, 4):                               # f1 variants, CC_PRESERVE_ORDER
        cc.coulomb_collide(torch.from_numpy(w.v).cuda(), torch.from_numpy(w.cell).cuda(), M, step=3, flags=fl,
                           **w.params())
    # f2 push, f3 recombination, f4 P2C, host-buffer entry
    x = torch.rand((3, n), dtype=torch.float64, device="cuda")
    g = cc.Grid(1, (M,), (1.0 / M,), 1)
    cc.cc_push(x, out2.v_out.clone(), out2.cell_out.clone(), g, dt=1e-10, perm=out2.perm_out, cells=M,
               E=torch.ones((3, M), dtype=torch.float64, device="cuda"))
    cc.cc_recombine(out2.v_out, out2.cell_out, torch.full((M,), 0.3, dtype=torch.float64, device="cuda"),
                    eps_bind=1e-18)
    cc.cc_p2c_moments(cc.cc_p2c(out.v_out, out.cell_out, M, sub=4))
    hb = cc.alloc_host_buffer(n, M, torch.device("cuda"))
    cc.coulomb_collide_host(torch.from_numpy(w.v), torch.from_numpy(w.cell), M, out_v=torch.empty((3, n),
                            dtype=torch.float64), out_cell=torch.empty(n, dtype=torch.int32), dev_buffer=hb,
                            **w.params())
torch.cuda.synchronize()
print("case ok")
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san_case.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
