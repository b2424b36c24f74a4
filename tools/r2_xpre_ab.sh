UCG_CROSS_PREFETCH=1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "fused or c2_small or c1_pipeline or graph or segment or many_partitions or full_vs_reference or fence_fused" > /tmp/p2.log 2>&1; echo "pytest xpre rc=$?"; tail -1 /tmp/p2.log
for rep in 1 2; do
for parts in 8 64; do
  for v in "R1" "UCG_CROSS_PREFETCH=0" "UCG_CROSS_PREFETCH=1" "UCG_CROSS_PREFETCH=1 UCG_ITEM_LOG2=11" "UCG_CROSS_PREFETCH=1 UCG_ITEM_LOG2=13"; do
    if [ "$v" = R1 ]; then (cd build/r1tree && timeout 600 python bench.py --parts $parts --no-engine-e2e --no-cpu-baseline --e2e-steps 1 --steps 40 > /tmp/m.json 2>/dev/null)
    else env $v timeout 600 python bench.py --parts $parts --no-engine-e2e --no-cpu-baseline --e2e-steps 1 --steps 40 --no-tuned-heap > /tmp/m.json 2>/dev/null; fi
    python -c "import json;d=json.loads(open('/tmp/m.json').read().strip().splitlines()[-1]);print('$v parts=$parts rep=$rep', round(d['ms_per_step']*1e3,2), round(d['roofline']['kernel_ms']*1e3,1), d['result'])"
  done
done
done
