import sys, numpy as np
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import paper_2507_11916_b200 as bida
from paper_2507_11916_b200.models import make_bmlp1
from oracle_lib import Oracle
o = Oracle()
blob = make_bmlp1("rc", hidden=[128, 128], classes=21, ensemble=1, seed=5)
p = bida.random_walks("rc", 300, 0, 30, seed=3)
with bida.MlpModelBackend("rc", blob, 0.5) as be:
    h, lg = be.evaluate_logits(p)
ho, lo = o.mlp_evaluate(blob, 100, 0.5, p, want_logits=True, E=1, Cc=21)
print("h equal:", (h == ho).all(), (h != ho).sum(), "logits equal:", np.array_equal(lg, lo))
print(h[:20], ho[:20])
print(lg[0, 0, :6], lo[0, 0, :6])
