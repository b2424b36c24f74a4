# Final 1-GPU pass after the top-trigger early mode (same steps as r2_final2.sh)
# GPU tests, smoke, every workload's bench line, the reference arm, the launch
# list and ncu captures of the fused C2 kernel and the Sobel kernel
D=gpurun_out/r2z3; mkdir -p $D
nvidia-smi -q -d POWER > $D/power_limits.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $D/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $D/n1.json 2> $D/n1.err; echo "c2 rc=$?"
for w in c1 c1lit c3 c4 c5 wc; do timeout 900 python bench.py --workload $w > $D/$w.json 2> $D/$w.err; echo "$w rc=$?"; done
timeout 600 python bench.py --parts 8 --no-engine-e2e --no-tuned-heap --no-cpu-baseline > $D/shard8.json 2> $D/shard8.err; echo "shard8 rc=$?"
timeout 1200 python bench.py --impl reference > $D/ref.json 2> $D/ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --steps 2 --warmup 3 --no-engine-e2e --no-cpu-baseline --no-tuned-heap > $D/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_segment_pass1 -s 5 -c 1 -o $D/ncu_fused python bench.py --steps 2 --warmup 3 --no-engine-e2e --no-cpu-baseline --no-tuned-heap > $D/ncu_full.log 2>&1; echo "ncu fused rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sobel_tma -c 1 -o $D/ncu_sobel python tools/sobel_time.py > $D/ncu_sobel.log 2>&1; echo "ncu sobel rc=$?"
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2z3/*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split('/')[-1], d.get("value"), d.get("unit"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"), (d.get("cpu_baseline") or {}).get("value"), (d.get("clocks") or {}).get("sm_mhz"))
    except Exception as e: print(f, "ERR", e)
P
