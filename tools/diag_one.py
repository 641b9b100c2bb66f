import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2108_13976_b200 as W
K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
kw = dict(num_taggers=3, num_runners=30, obs_mode=1, k_nearest=K, grid_size=50, seed=9)
oc = O.make_config(**kw)
dc = W.TagConfig(**{f: getattr(oc, f) for f, _ in O.TagConfigC._fields_})
ws = W.Workspace(dc, 1)
o = O.OracleWorld(oc, 1)
dev = ws.store.pull("observations"); ora = o.pull("observations")
print("loc equal", np.array_equal(ws.store.pull("loc_x"), o.pull("loc_x")), np.array_equal(ws.store.pull("loc_y"), o.pull("loc_y")))
bad = np.argwhere(dev != ora)
print("mismatches", len(bad))
for a in range(3):
    print("agent", a)
    print(" dev", np.round(dev[0, a], 3).tolist())
    print(" ora", np.round(ora[0, a], 3).tolist())
