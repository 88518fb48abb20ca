#!/bin/bash
# bench sweep: TAG "config:args;config:args;..."
TAG=$1
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
if [ -n "$3" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$3" > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
fi
IFS=';' read -ra RUNS <<< "$2"
i=0
for r in "${RUNS[@]}"; do
  c=${r%%:*}; args=${r#*:}
  echo "== $c $args" >> $O/${TAG}_sweep.txt
  timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e $args > $O/${TAG}_run$i.json 2> $O/${TAG}_run$i.err
  python -c "
import json
d=json.load(open('$O/${TAG}_run$i.json'))
print(round(d['ms_per_step'],3), {k:v['ms'] for k,v in d['stages'].items()}, 'grouping', d['counters'].get('grouping'))
" >> $O/${TAG}_sweep.txt 2>&1
  i=$((i+1))
done
echo done > $O/${TAG}_done
