import cProfile, pstats, io, sys, tempfile
sys.path.insert(0, '.')
import torch
from paper_2511_23030_b200.workloads import build_c2
eng = build_c2(1_000_000, 16, store_dir=tempfile.mkdtemp())
eng.warm_graphs()
for s in range(20):
    eng.optimization_step(0, s)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for s in range(300):
    eng.optimization_step(1, s)
torch.cuda.synchronize()
pr.disable()
buf = io.StringIO()
pstats.Stats(pr, stream=buf).sort_stats("tottime").print_stats(45)
print(buf.getvalue())
