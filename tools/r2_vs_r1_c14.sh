for rep in 1 2; do
  for w in c1 c4; do
    for t in r1 r2; do
      if [ $t = r1 ]; then d=build/r1tree; else d=.; fi
      (cd $d && timeout 600 python bench.py --workload $w > /tmp/w.json 2>/dev/null)
      python -c "
import json
d=json.loads(open('/tmp/w.json').read().strip().splitlines()[-1]); print('$t $w rep=$rep', '%.4g' % d['value'], d['unit'], round(d['ms_per_step'],4))" 2>&1 | tail -1
    done
  done
done
