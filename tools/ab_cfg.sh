#!/bin/bash
# A/B of library environment knobs on one config (per-role breakdown): tools/ab_cfg.sh cfg5p "X=1" "X=2"
cfg=$1; shift
for setting in "$@"; do
  echo "$setting: $(env $setting timeout 300 python tools/prof_configs.py $cfg 2>&1 | tail -1 | cut -c1-420)"
  env $setting timeout 300 python - <<PY
import os, sys, torch
sys.path.insert(0, ".")
import paper_2407_14801_b200 as sq, sqinputs as S
kind, n, seed = S.CONFIGS["$cfg"]
k, v = S.generate(kind, n, seed)
kd = torch.from_numpy(k).cuda(); vd = torch.from_numpy(v).cuda() if v is not None else None
ts = []
for i in range(6):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wk = kd.clone(); wv = vd.clone() if vd is not None else None
    torch.cuda.synchronize(); a.record()
    if wv is not None: sq.sort_pairs_u32_u32(wk, wv, seed)
    elif k.dtype.name == "uint64": sq.sort_u64(wk, seed)
    else: sq.sort_u32(wk, seed)
    b.record(); torch.cuda.synchronize()
    if i: ts.append(a.elapsed_time(b))
print("   $setting ms", sorted(ts)[len(ts)//2])
PY
done
