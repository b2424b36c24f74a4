# After the start-ticket ordering fix: the whole GPU suite (incl. long step
# chains, and the sharded chains at N ranks), then top vs late trigger at the
# 8-GPU shard size and C2 over N ranks, 5 alternating reps
N=$(nvidia-smi -L | wc -l)
D=gpurun_out/r2f; mkdir -p $D
timeout 1800 python -m pytest tests -q -m gpu > $D/pytest_gpu_n$N.log 2>&1; echo "pytest rc=$?"; tail -3 $D/pytest_gpu_n$N.log
for rep in 1 2 3 4 5; do
  for e in "X=0" "UCG_EARLY_LATE_TRIGGER=1"; do
    tag=$(echo $e | tr '=' '_')
    env $e timeout 600 python bench.py --gpus $N --parts $((8 * N)) --no-engine-e2e --no-tuned-heap --no-cpu-baseline > $D/s8_n${N}_${tag}_$rep.json 2> $D/s8_n${N}_${tag}_$rep.err; echo "s8 $tag $rep rc=$?"
    env $e timeout 600 python bench.py --gpus $N --no-engine-e2e --no-tuned-heap --no-cpu-baseline > $D/c2_n${N}_${tag}_$rep.json 2> $D/c2_n${N}_${tag}_$rep.err; echo "c2 $tag $rep rc=$?"
  done
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2f/*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split('/')[-1], d.get("n_gpus"), round(d.get("value")/1e9,2), round(d.get("ms_per_step")*1e3,2), (d.get("parity") or {}).get("result_match"))
    except Exception as e: print(f, "ERR", e)
P
