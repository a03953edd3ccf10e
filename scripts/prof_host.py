"""Host-side profile of an adaptive run (cProfile) next to its device time.

usage: prof_host.py {c0|c2} [t_final]
"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2108_13622_b200 as xb  # noqa: E402
from paper_2108_13622_b200 import leja, scenarios as sc  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c0"
if which == "c3":
    mk = lambda tf=None: sc.kh_setup(4096, tol=1e-5, t_final=1e9, max_accepted=(2 if tf else 20))  # noqa: E731
    scheme = xb.Scheme.EXPRB43
elif which == "c0":
    mk = lambda tf=None: sc.kh_setup(128) if tf is None else sc.kh_setup(128, t_final=tf)  # noqa: E731
    scheme = xb.Scheme.EXPRB43
else:
    mk = lambda tf=None: sc.harris_setup(512) if tf is None else sc.harris_setup(512, t_final=tf)  # noqa: E731
    scheme = xb.Scheme.EXPRB54S4
tf = float(sys.argv[2]) if len(sys.argv) > 2 else None
s = mk(tf)
xb.run(xb.RunConfig(scenario=mk(0.02), scheme=scheme, tol=s.tol,
                    max_accepted=mk(0.02).max_accepted))   # warm
leja._coeff_cache.clear()
torch.cuda.synchronize()
t0 = time.perf_counter()
rep = xb.run(xb.RunConfig(scenario=s, scheme=scheme, tol=s.tol, max_accepted=s.max_accepted))
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print(f"{which}: wall {wall:.4f} s, {rep.accepted} accepted, {rep.rhs_evals} rhs, "
      f"{wall / max(rep.accepted, 1) * 1e3:.3f} ms/step, "
      f"{wall / rep.rhs_evals * 1e6:.1f} us/rhs", flush=True)
leja._coeff_cache.clear()
pr = cProfile.Profile()
pr.enable()
rep = xb.run(xb.RunConfig(scenario=s, scheme=scheme, tol=s.tol, max_accepted=s.max_accepted))
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
pstats.Stats(pr).sort_stats("cumtime").print_stats(30)
