import sys, time, torch
sys.path.insert(0, ".")
import paper_2404_11631_b200 as p
from paper_2404_11631_b200.instances import gen_meanvar_instance
from paper_2404_11631_b200.tasks import MeanVarProblem, MvFwEngine
b = p.make_backend("cuda")
prob = MeanVarProblem(gen_meanvar_instance(1000, p.RngStream(42, 0)), b)
prob.resample(p.RngStream(42, 2), 10_000)
eng = MvFwEngine(prob, 25, 4096)
ss = prob.sample_set
eng.q = torch.empty(10_000, dtype=torch.float64, device="cuda")
def ev(fn, n=5):
    torch.cuda.synchronize(); t = time.perf_counter()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / n, (time.perf_counter() - t) * 1e3 / n
eager = lambda: eng._steps(eng.rings[0], ss.samples, ss.mean, 10_000)
print("eager (gpu ms, host ms):", ev(eager))
torch.cuda.cudart().cudaProfilerStart()
eager()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
# kernel-only breakdown: single kernels
x, mean, q = ss.samples, ss.mean, eng.q
w = eng.rings[0][0]
print("matvec:", ev(lambda: b.matvec_device(x, w, out=q, center=mean), 20))
print("matvec_t:", ev(lambda: b.matvec_t_device(x, q, out=eng.gq, center=mean), 20))
print("tree_sums2:", ev(lambda: p._lib.call("simopt_tree_sums2", p._lib.stream_ptr(), p._lib.ptr(q), p._lib.ptr(q), 10000, p._lib.ptr(eng.quad), p._lib.ptr(w), p._lib.ptr(mean), 1000, p._lib.ptr(eng.lin), 4096), 20))
