"""A/B kernel timing for tuning: per-kernel device ms of one config for several builds of the library.

python tools/dev/ab_bench.py CONFIG REPS LIB[@VAR=VAL,...] [...]   (run on the GPU box; alternates the
libraries in fresh subprocesses, 3 rounds, prints the per-kernel median ms per multiply of each; the
optional @VAR=VAL list sets environment knobs of that run, e.g. lib.so@GF2X_BOT_B=6)
"""
import json
import os
import statistics
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def child(cfg, reps, lib):
    import numpy as np
    import torch
    import paper_1708_09746_b200 as G
    from gf2x_synth import CONFIGS, batch_pair, operand_pair
    G.load(lib)
    bits, batch = CONFIGS[cfg]
    a, b = operand_pair(bits) if batch == 1 else batch_pair(bits, batch)
    da = torch.from_numpy(a.reshape(-1).view(np.int64)).cuda().view(torch.uint64)
    db = torch.from_numpy(b.reshape(-1).view(np.int64)).cuda().view(torch.uint64)
    c = torch.empty(batch * (2 * ((bits + 63) // 64)), dtype=torch.uint64, device="cuda")
    for it in range(2):
        if it == 1:
            G.profile_enable(True)
        for _ in range(reps if it else 3):
            G.gf2x_mul_batched(da, bits, db, bits, batch, c)
        torch.cuda.synchronize()
    rep = G.profile_report()
    print(json.dumps({r["kernel"]: r["ms"] / reps for r in rep}))


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]), sys.argv[4])
        sys.exit(0)
    cfg, reps, libs = sys.argv[1], sys.argv[2], sys.argv[3:]
    res = {l: [] for l in libs}
    for _ in range(3):
        for l in libs:
            path, _, knobs = l.partition("@")
            env = dict(os.environ, **dict(kv.split("=", 1) for kv in knobs.split(",") if kv))
            out = subprocess.run([sys.executable, __file__, "--child", cfg, reps, path], capture_output=True, text=True,
                                 env=env)
            if out.returncode:
                print(out.stderr[-2000:])
                sys.exit(1)
            res[l].append(json.loads(out.stdout.strip().splitlines()[-1]))
    for l in libs:
        ks = res[l][0].keys()
        med = {k: round(statistics.median(r[k] for r in res[l]), 4) for k in ks}
        print(os.path.basename(l).replace(' ', ''), round(sum(med.values()), 4), med)
