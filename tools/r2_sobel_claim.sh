# Sobel tile claiming A/B (claimed tiles with the self-resetting claim pair vs
# round-robin tiles), same box, alternating; full GPU tests; ncu; C4 line
D=gpurun_out/r2u; mkdir -p $D
timeout 1500 python -m pytest tests -q -m gpu -x > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?"
for rep in 1 2 3 4; do
  for st in "X=0" "UCG_SOBEL_STATIC=1"; do
    env $st timeout 120 python tools/sobel_time.py | sed "s/^/{\"static\": \"$st\", \"rep\": $rep, \"line\": /; s/$/}/" >> $D/ab.jsonl
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sobel_tma -c 1 -o $D/ncu_tma_claim python tools/sobel_time.py > $D/ncu_tma_claim.log 2>&1; echo "ncu rc=$?"
timeout 600 python bench.py --workload c4 > $D/c4.json 2> $D/c4.err; echo "c4 rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 $D/pytest_gpu.log
cat $D/ab.jsonl
