"""Edit statistics of the graph step's incremental binning (development tool).

python tools/incstat.py
Runs 600 graph-replayed fit() steps of configs 3 and 2 and prints, per
20-step window, the most list edits (nops) and changed Gaussians a step
produced, plus the number of graph captures (an edit-capacity overflow
re-captures).  Sized the capacities _CHG_CAP / kOpsCap.
"""
import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2603_09621_b200 as gs
from paper_2603_09621_b200 import synth
for cfg in (3, 2):
    p = synth.make_problem(synth.CONFIGS[cfg])
    f = gs.GaussianField(*p["field"])
    lr = gs.Volume(p["lr_grid"], p["lr"])
    step = gs.TrainStep(lr, gs.RenderOptions(), (8, 8, 4), "l1")
    state = gs.AdamState.create(f)
    lrs = gs.FitConfig().resolved_lrs(p["lr_grid"].spacing)
    rows = []
    for it in range(600):
        step.step(f, state, lrs)
        b = step._graph.bufs
        rows.append((int(b["nops"].item()), int(b["chg_count"].item()), int(b["overflow"].item())))
    caps = step.graph_captures
    nops = [r[0] for r in rows]
    chg = [r[1] for r in rows]
    print("config", cfg, "captures", caps, "max nops", max(nops), "max pending chg", max(chg))
    print(" nops per 20 steps (max):", [max(nops[i:i+20]) for i in range(0, 600, 20)])
    print(" chg per 20 steps (max):", [max(chg[i:i+20]) for i in range(0, 600, 20)])
    print(" overflow steps:", [i for i, r in enumerate(rows) if r[2]])
