# same-box A/B of the round-1 build (build/r1tree, commit 79d596b) against the
# current one: the C1 step (latency-bound) and the C2 shard / full sizes
for rep in 1 2 3; do
  echo "== rep $rep"
  echo -n "r2 "; python tools/c1_probe.py 2>&1 | grep -E "kernels:|graph of 32"
  (cd build/r1tree && echo -n "r1 " && python tools/c1_probe.py 2>&1 | grep -E "kernels:|graph of 32")
done
for rep in 1 2; do
for parts in 8 64; do
  timeout 600 python bench.py --parts $parts --no-engine-e2e --no-cpu-baseline --e2e-steps 1 --steps 40 > gpurun_out/r2s.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2s.json').read().strip().splitlines()[-1]);print('r2 parts=$parts', round(d['ms_per_step']*1e3,2))"
  (cd build/r1tree && timeout 600 python bench.py --parts $parts --no-engine-e2e --no-cpu-baseline --e2e-steps 1 --steps 40 > ../../gpurun_out/r1s.json 2>/dev/null)
  python -c "import json;d=json.loads(open('gpurun_out/r1s.json').read().strip().splitlines()[-1]);print('r1 parts=$parts', round(d['ms_per_step']*1e3,2))"
done
done
