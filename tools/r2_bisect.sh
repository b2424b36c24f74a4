# same-box A/B: round-1 build, the safety-fix commit, the tagged-tail commit, current
for rep in 1 2; do
  for t in r1tree tree_be32b64 tree_394fe52 .; do
    if [ "$t" = "." ]; then d=.; else d=build/$t; fi
    k=$(cd $d && python tools/c1_probe.py 2>&1 | grep -E "kernels:" | awk '{print $NF}')
    (cd $d && timeout 600 python bench.py --parts 64 --no-engine-e2e --no-cpu-baseline --e2e-steps 1 --steps 30 > /tmp/b64.json 2>/dev/null)
    (cd $d && timeout 600 python bench.py --parts 8 --no-engine-e2e --no-cpu-baseline --e2e-steps 1 --steps 40 > /tmp/b8.json 2>/dev/null)
    python -c "
import json
a=json.loads(open('/tmp/b64.json').read().strip().splitlines()[-1]); b=json.loads(open('/tmp/b8.json').read().strip().splitlines()[-1])
print('$t rep=$rep c1_kernel=$k p64=%.2f p8=%.2f' % (a['ms_per_step']*1e3, b['ms_per_step']*1e3))"
  done
done
