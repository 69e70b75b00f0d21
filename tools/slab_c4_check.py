"""C4-size check of the x-slab path at world size 1 (edge + interior parts,
two streams, periodic self-exchange) against the single-domain sweep, bitwise."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1507_06565_b200 as pg
from paper_1507_06565_b200 import configs
from paper_1507_06565_b200.dist import SlabSimulation

w = configs.c4()
g = w.geometry()
sim = configs.make_simulation(w, g)
sim.step(7)
a = sim.get_pdfs()
del sim
ss = SlabSimulation(w, 0, 1, device=0, geometry=None)
ss.step(7)
b = ss.sim.get_pdfs()
fl = g.flags.reshape(w.dims[::-1]) == 0
eq = np.array_equal(a[:, fl], b[:, fl])
print("C4 slab(world 1) == single domain after 7 steps:", eq)
if not eq:
    d = a[:, fl] != b[:, fl]
    print("differing slots:", int(d.sum()), "of", d.size)
