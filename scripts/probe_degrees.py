"""Leja degree of every phi-action of an adaptive run (config 3 / 4), and how
many of them end on an odd term (the lookahead schedule then spends one more
launch to resolve the residual).

usage: probe_degrees.py {3|4} [steps]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13622_b200 as xb  # noqa: E402
from paper_2108_13622_b200 import integrators, leja, scenarios as sc  # noqa: E402

which = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
s = sc.CONFIGS[which]()
s.max_accepted = steps
degs = []
orig = leja.apply_phi_leja


def logged(l, matvec, v, dt, shift, tol):
    r = orig(l, matvec, v, dt, shift, tol)
    degs.append((l, r.iterations))
    return r


integrators.apply_phi_leja = logged
scheme = xb.Scheme.EXPRB54S4 if which == 4 else xb.Scheme.EXPRB43
rep = xb.run(xb.RunConfig(scenario=s, scheme=scheme, tol=s.tol, max_accepted=steps))
hist = collections.Counter(d for _, d in degs)
odd = sum(1 for _, d in degs if d & 1)
print(f"config {which}: {len(degs)} phi-actions in {rep.accepted} steps, degrees {sorted(hist.items())}, "
      f"{odd} end on an odd term; total terms {sum(d for _, d in degs)}")
