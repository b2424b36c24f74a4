# Sobel arithmetic A/B (fp16-subnormal vs integer) for the tiled and the
# row-streaming kernels, same box, alternating; parity test; ncu of each
D=gpurun_out/r2s; mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "sobel" > $D/pytest_sobel.log 2>&1; echo "pytest rc=$?"
for rep in 1 2 3; do
  for v in 1 0; do for a in int half; do
    UCG_SOBEL_VARIANT=$v UCG_SOBEL_ARITH=$a timeout 120 python tools/sobel_time.py | sed "s/^/{\"arith\": \"$a\", \"rep\": $rep, \"line\": /; s/$/}/" >> $D/ab.jsonl
  done; done
done
for a in half int; do
  UCG_SOBEL_ARITH=$a timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sobel_tma -c 1 -o $D/ncu_tma_$a python tools/sobel_time.py > $D/ncu_tma_$a.log 2>&1; echo "ncu $a rc=$?"
done
UCG_SOBEL_VARIANT=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sobel_rows -c 1 -o $D/ncu_rows_half python tools/sobel_time.py > $D/ncu_rows_half.log 2>&1; echo "ncu rows rc=$?"
timeout 600 python bench.py --workload c4 > $D/c4.json 2> $D/c4.err; echo "c4 rc=$?"
cat $D/ab.jsonl
