"""One launch of each non-partition kernel for ncu captures: K2 evaluate (config 2, 64
assignments), K7 levels and assigned makespan (config 2), K8 DES (config-5 batch of 1024
simulations), the exact 2-way FM batch (gp partitions), and the device transpose."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1502_07451_b200 as H
from paper_1502_07451_b200 import kway
from paper_1502_07451_b200.csr import DagCSR
from paper_1502_07451_b200.sim import MachineModel, simulate_batch
from paper_1502_07451_b200.policies import DmdaPolicy, gp_build_batch

c2 = kway.layered_dag(100_000, 1_000_000, seed=0)
ew, nw = kway.integer_weights(c2.w_xfer), kway.integer_weights(c2.w_gpu)
r = kway.partition_kway(kway.symmetrize(c2, ew, nw), 8, tol=0.03)
parts = kway.kernel_to_node_parts(c2, r.part).unsqueeze(0).repeat(64, 1).contiguous()
kway.evaluate_batch(c2, parts, 8, nw.to(torch.int64))
kway.levels(c2)
kway.assigned_makespan(c2, parts[0].contiguous(), k=8)
DagCSR.from_out_csr(c2.root, c2.out_ptr, c2.out_dst)
model = H.SyntheticCostModel()
graphs = [H.attach_weights(H.generate_random_dag(38, 75, "MA", 1024, seed=i), model)
          for i in range(1024)]
gp = gp_build_batch(graphs)
simulate_batch(graphs, [DmdaPolicy()] * len(graphs), MachineModel(3, 1), validate_graphs=False)
torch.cuda.synchronize()
print("ok")
