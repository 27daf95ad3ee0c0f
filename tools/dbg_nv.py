import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2404_11631_b200 as pkg
from paper_2404_11631_b200.tasks import NewsvendorProblem, NewsvendorTask
from oracle import oracle as orc
g = dict(np.load("tests/golden/newsvendor.npz"))
t = NewsvendorTask(unit_cost=g["unit_cost"], holding_cost=g["holding_cost"], selling_value=g["selling_value"], demand_mean=g["demand_mean"], demand_std=g["demand_std"], budget_costs=g["budget_costs"], budget=float(g["budget"][0]))
prob = NewsvendorProblem(t, pkg.make_backend("cuda"))
prob.resample(pkg.RngStream(42, 2), 301)
got = prob.gradient(g["xq"])
cnt = prob.dev.counts(torch.from_numpy(g["xq"]).cuda()).cpu().numpy()
want_cnt = orc.ecdf_counts(g["demands"], g["xq"])
print("counts equal", np.array_equal(cnt, want_cnt), cnt[:6], want_cnt[:6])
bad = np.flatnonzero(got != g["grad"])
print("bad", bad, got[bad], g["grad"][bad])
print("oracle grad eq", np.array_equal(orc.nv_gradient_hat(g["xq"], g["demands"], g["unit_cost"], g["holding_cost"], g["selling_value"]), g["grad"]))
