#!/bin/bash
# GPU box: small-n latencies, then ncu launch lists of replayed small levels (2^16, 2^20).
mkdir -p gpurun_out
python tools/small_n.py 2>&1 | tee gpurun_out/small_n.jsonl | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['n'], d['ok'], d['median_ms'], d['min_ms'], d['stats']['kernel_launches'])
"
for lg in ${SIZES:-16 18 20}; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/small_launches_$lg.csv \
    python tools/small_once.py $lg > gpurun_out/small_ncu_$lg.log 2>&1
  python - <<PY
import csv, re
rows = [r for r in csv.reader(open("gpurun_out/small_launches_$lg.csv")) if len(r) > 14 and r[0].isdigit()]
ks = [(re.sub(r"\(.*", "", r[4]).replace("void sq::", "").replace("sq::", "")[:48], r[7], r[8], float(r[14].replace(",", "")) / 1e3) for r in rows if "sq::" in r[4]]
per = len(ks) // 5
last = ks[-per:]
print("2^$lg: kernels per replayed call", per, "sum us", round(sum(k[3] for k in last), 1))
for k in last: print("   ", k[0], k[1], k[2], round(k[3], 1))
PY
done
