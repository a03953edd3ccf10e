import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import paper_2108_13622_b200 as xb
from paper_2108_13622_b200 import scenarios as sc
s = sc.harris_setup(512, t_final=1.0)
xb.run(xb.RunConfig(scenario=sc.harris_setup(512, t_final=0.05), scheme=xb.Scheme.EXPRB54S4, tol=1e-6))
pr = cProfile.Profile(); pr.enable()
t0=time.perf_counter()
rep = xb.run(xb.RunConfig(scenario=s, scheme=xb.Scheme.EXPRB54S4, tol=1e-6))
print("wall", time.perf_counter()-t0, rep.accepted, rep.rhs_evals)
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(25)
