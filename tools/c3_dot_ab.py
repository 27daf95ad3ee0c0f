"""A/B of the fused Newton-CG scalars: one-CTA dot (default) vs the fixed-tree dot (SIMOPT_CG_TREE=1), C3 bit-packed."""
import os, sys, time, statistics
import torch
sys.path.insert(0, ".")
import paper_2404_11631_b200 as p
from paper_2404_11631_b200.newton import newton_cg
from paper_2404_11631_b200.sampling import synth_classification
from paper_2404_11631_b200.tasks import LogisticTask
b = p.make_backend("cuda")
task = LogisticTask(synth_classification(1000, p.RngStream(42, 0), n_rows=1_000_000, packed=True))
res = {"fast": [], "tree": []}
for rep in range(4):
    for mode in ("fast", "tree"):
        os.environ["SIMOPT_CG_TREE"] = "1" if mode == "tree" else "0"
        newton_cg(task, 2, 10, b); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); newton_cg(task, 10, 10, b); e1.record(); torch.cuda.synchronize()
        res[mode].append(e0.elapsed_time(e1) / 10)
for k, v in res.items():
    print(k, "ms per Newton iteration", round(statistics.median(v), 4), [round(x, 4) for x in v])
