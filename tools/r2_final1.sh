# round-2 measurement pass on one GPU: every workload's bench line, the
# reference arm on the full C2 config, the launch list and ncu captures
mkdir -p gpurun_out/r2h
timeout 600 python bench.py > gpurun_out/r2h/n1.json 2> gpurun_out/r2h/n1.err; echo "c2 rc=$?"
for w in c1 c1lit c3 c4 c5 wc; do timeout 600 python bench.py --workload $w > gpurun_out/r2h/$w.json 2> gpurun_out/r2h/$w.err; echo "$w rc=$?"; done
timeout 1800 python bench.py --impl reference > gpurun_out/r2h/ref.json 2> gpurun_out/r2h/ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2h/launches.csv python bench.py --steps 2 --warmup 3 --no-engine-e2e --no-cpu-baseline > gpurun_out/r2h/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_segment_pass1 -s 5 -c 1 -o gpurun_out/r2h/ncu_fused python bench.py --steps 2 --warmup 3 --no-engine-e2e --no-cpu-baseline > gpurun_out/r2h/ncu_full.log 2>&1; echo "ncu fused rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_word_flags -c 1 -o gpurun_out/r2h/ncu_wordflags python bench.py --workload wc --steps 2 --warmup 3 > gpurun_out/r2h/ncu_wc.log 2>&1; echo "ncu wc rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sobel_tma -c 1 -o gpurun_out/r2h/ncu_sobel python tools/sobel_time.py > gpurun_out/r2h/ncu_sobel.log 2>&1; echo "ncu sobel rc=$?"
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2h/*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("value"), d.get("unit"), (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"), (d.get("cpu_baseline") or {}).get("value"))
    except Exception as e: print(f, "ERR", e)
P
