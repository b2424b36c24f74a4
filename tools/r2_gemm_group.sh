# GEMM raster group size A/B (UCG_GEMM_GROUP, m-blocks per group of the CTA-pair kernel)
D=gpurun_out/r2gg; mkdir -p $D
for g in 8 4; do UCG_GEMM_GROUP=$g timeout 900 python -m pytest tests/test_gpu_gemm.py -q -m gpu > $D/pytest_g$g.log 2>&1; echo "pytest g$g rc=$?"; tail -1 $D/pytest_g$g.log; done
for rep in 1 2; do for g in 16 8 4 32; do
  UCG_GEMM_GROUP=$g timeout 300 python tools/gemm_f32_perf.py | sed "s/^/{\"group\": $g, \"rep\": $rep, \"line\": /; s/$/}/" >> $D/perf.jsonl
done; done
for rep in 1 2; do for g in 16 8; do
  UCG_GEMM_GROUP=$g timeout 900 python bench.py --workload c5 > $D/c5_g${g}_$rep.json 2> $D/c5_g${g}_$rep.err
done; done
for g in 16 8; do
  UCG_GEMM_GROUP=$g timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_gemm_tf32_2sm -c 2 python tools/gemm_f32_perf.py > $D/ncu_g$g.txt 2>&1; echo "ncu g$g rc=$?"
done
cat $D/perf.jsonl
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2gg/c5_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f.split('/')[-1], round(d["value"]/1e12,1), round(d["ms_per_step"],2), d["clocks"]["sm_mhz"])
P
grep -E 'k_gemm|dram__bytes|gpu__time' $D/ncu_g16.txt $D/ncu_g8.txt | head -20
