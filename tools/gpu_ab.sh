#!/bin/bash
# A/B of an environment toggle on bench lines: configs in $3 (default "scale text"),
# each run $4 times (default 3) alternating VAR=1 / VAR=0 ($2, e.g. GAKCO_PDL)
O=gpurun_out; T=${1:-ab}; V=${2:-GAKCO_PDL}; C=${3:-scale text}; R=${4:-3}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
for c in $C; do
  for r in $(seq 1 $R); do
    for v in 1 0; do
      env $V=$v timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e --config $c \
        > $O/${T}_${c}_${v}_$r.json 2> $O/${T}_${c}_${v}_$r.err
    done
  done
done
python - "$O" "$T" "$C" "$R" > $O/${T}_summary.txt <<'EOF'
import json, sys
O, T, C, R = sys.argv[1], sys.argv[2], sys.argv[3].split(), int(sys.argv[4])
for c in C:
    for v in ("1", "0"):
        ms = []
        for r in range(1, R + 1):
            try:
                ms.append(json.load(open(f"{O}/{T}_{c}_{v}_{r}.json"))["ms_per_step"])
            except Exception as e:
                ms.append(f"err {e}")
        print(c, v, ms)
EOF
echo done > $O/${T}_done
