python -c "import __graft_entry__ as g; g.build()" || exit 1
for m in warm steady cold; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_collide_large" -s 3 -c 1 -o gpurun_out/r03e_$m python tools/prof_modes.py $m 4 > gpurun_out/r03e_$m.log 2>&1; echo $m rc=$?
done
