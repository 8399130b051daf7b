import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import torch
from paper_1502_07451_b200 import gen
from paper_1502_07451_b200.policies import gp_pins_batch
b = gen.RandomDagFactory(38, 75, "MA", 1024).batch(range(4096))
gp_pins_batch(b); torch.cuda.synchronize()
b = gen.RandomDagFactory(38, 75, "MA", 1024).batch(range(4096))
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter(); gp_pins_batch(b); torch.cuda.synchronize(); t1 = time.perf_counter()
pr.disable()
print("gp_pins_batch s", t1 - t0)
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
