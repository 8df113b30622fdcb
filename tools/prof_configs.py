"""Per-kernel-role breakdown (library CUDA events, sq_profile) of one sort of each
named config: where the time of the non-headline configs goes."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_14801_b200 as sq
import sqinputs as S

names = sys.argv[1:] or ["cfg3", "cfg4_swapped", "cfg4_sorted", "cfg5p"]
for name in names:
    kind, n, seed = S.CONFIGS[name]
    k, v = S.generate(kind, n, seed)
    kd = torch.from_numpy(k).cuda()
    vd = torch.from_numpy(v).cuda() if v is not None else None
    def run():
        if vd is not None:
            sq.sort_pairs_u32_u32(kd.clone(), vd.clone(), seed)
        elif k.dtype.name == "uint64":
            sq.sort_u64(kd.clone(), seed)
        else:
            sq.sort_u32(kd.clone(), seed)
    run(); torch.cuda.synchronize()
    sq.profile(True); sq.profile_read(); run(); torch.cuda.synchronize(); sq.profile(False)
    prof = {r: [c, round(ms, 3)] for r, (c, ms) in sq.profile_read().items()}
    print(name, json.dumps(sq.get_stats()), json.dumps(prof), flush=True)
