timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2k_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2k_pytest.log
for rep in 1 2; do
for t in 1 0; do
  for parts in 8 64; do
    UCG_TAGGED_TAIL=$t timeout 600 python bench.py --parts $parts --no-engine-e2e --no-cpu-baseline --e2e-steps 1 --steps 50 > gpurun_out/r2k_tail${t}_p${parts}_r$rep.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/r2k_tail${t}_p${parts}_r$rep.json').read().strip().splitlines()[-1]);print('tagged=$t parts=$parts rep=$rep', round(d['ms_per_step']*1e3,2), 'us/step kernel', round(d['roofline']['kernel_ms']*1e3,2), d['parity'] and d['parity']['result_match'], d['result'])"
  done
done
done
