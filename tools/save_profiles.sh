#!/bin/bash
# Copy one tools/r02_refresh.sh run from gpurun_out/ into profiles/ under a tag.
set -eu
tag=$1
g=gpurun_out; p=profiles
cp $g/bench_full.json $p/${tag}_bench.json
cp $g/launches.csv $p/${tag}_launches.csv
calls=$(python - <<PY
import csv
rows=list(csv.reader(open("$g/launches.csv"))); hdr=None; ids=set()
for r in rows:
    if r and r[0]=="ID": hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if "k_transpose" in d["Kernel Name"]: ids.add(d["ID"])
print(len(ids))
PY
)
python tools/summarize_launches.py $g/launches.csv $p/${tag}_launches.md $p/ncu_traffic.json $calls > /dev/null
{ echo "# ${tag}: ncu --set full captures (first launch of each kernel in one cfg5 sort; tools/ncu_full.sh)"; echo
  echo "Cold-cache, serialised replays: use shares and ratios, not absolute times."; echo
  for k in k_colsort k_transpose_ws k_bucketsort; do
    [ -f $g/full_$k.md ] && sed '1d' $g/full_$k.md
    [ -f $g/full_${k}_lines.txt ] && { echo '```'; head -25 $g/full_${k}_lines.txt; echo '```'; echo; }
  done; } > $p/${tag}_ncu_full.md
[ -f $g/configs.log ] && grep -A20 "^| config" $g/configs.log > $p/${tag}_configs.md || true
[ -f $g/small_n.jsonl ] && cp $g/small_n.jsonl $p/${tag}_small_n.jsonl || true
[ -f $g/prof_configs.log ] && cp $g/prof_configs.log $p/${tag}_prof_configs.log || true
ls $p/${tag}_*
