timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "fused or c2_small or c1_pipeline or graph or tagged or fence_fused or full_vs_reference" > gpurun_out/r2o_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2o_pytest.log
for rep in 1 2; do
for v in "UCG_CHUNK_TAIL=0" "UCG_CHUNK_TAIL=1" "UCG_CHUNK_TAIL=1 UCG_CTAIL_ITEMS=592" "UCG_CHUNK_TAIL=1 UCG_CTAIL_ITEMS=148"; do
  for parts in 8 64; do
    env $v timeout 600 python bench.py --parts $parts --no-engine-e2e --no-cpu-baseline --e2e-steps 1 --steps 40 > gpurun_out/r2o_ab.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/r2o_ab.json').read().strip().splitlines()[-1]);print('$v parts=$parts rep=$rep', round(d['ms_per_step']*1e3,2), 'us/step', d['result'], (d.get('parity') or {}).get('result_match'))"
  done
done
done
