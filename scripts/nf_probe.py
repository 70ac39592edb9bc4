"""Run the cfg-3 near-field correction (K3) once for timing / ncu."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_00995_b200 as g

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10242
m = g.perturb_radial(g.build_sphere(n, 1.0), 2, 0.02)
dom = g.make_domain(m, 6)
p0 = g.make_fem(m, "P0")
nf = g.NearField(dom, dom, p0, "[1/r]", p0)
for it in range(2):
    torch.cuda.synchronize()
    t = time.time()
    nf.compute(0)
    torch.cuda.synchronize()
    print("pairs/entries", nf.info(), "calls", nf.stats()[0], "ms %.2f" % ((time.time() - t) * 1e3))
