"""One 456-wide diagonal block (config 5's supernode width) through block_ldlt:
the 16-CTA cluster BK (dev aid for the ncu capture of bk_cluster_kernel<16>)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2002_05018_b200 as d

n = int(os.environ.get("N", "456"))
rng = np.random.default_rng(456)
G = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2 * n)
M = (G + G.T) / 2
M[np.diag_indices(n)] += rng.uniform(-2, 2, n)
K = d.from_blocks([n], [(0, 0, M)])
plan = d.symbolic_factor(d.clique_graph(K), d.identity_ordering(1), K.sizes)
for _ in range(3):
    F = d.block_ldlt(K, plan)
torch.cuda.synchronize()
print("n", n, "n2x2", F.stats.n_2x2_pivots, "growth", F.stats.growth_factor)
