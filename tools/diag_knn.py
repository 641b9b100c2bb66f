"""Diagnostic: device vs oracle registration obs for a few K / A combos."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2108_13976_b200 as W
for kw, envs in [(dict(num_taggers=3, num_runners=30, obs_mode=1, k_nearest=20, grid_size=50, seed=9), 9),
                 (dict(num_taggers=3, num_runners=30, obs_mode=1, k_nearest=8, grid_size=50, seed=9), 9),
                 (dict(num_taggers=3, num_runners=30, obs_mode=1, k_nearest=9, grid_size=50, seed=9), 9),
                 (dict(num_taggers=3, num_runners=30, obs_mode=1, k_nearest=20, grid_size=8, seed=9), 9),
                 (dict(num_taggers=10, num_runners=90, obs_mode=1, k_nearest=20, grid_size=50, seed=9), 3)]:
    oc = O.make_config(**kw)
    dc = W.TagConfig(**{f: getattr(oc, f) for f, _ in O.TagConfigC._fields_})
    ws = W.Workspace(dc, envs)
    o = O.OracleWorld(oc, envs)
    dev = ws.store.pull("observations"); ora = o.pull("observations")
    bad = np.argwhere(dev != ora)
    print(kw, "geometry", ws.plan.geometry(), "mismatches", len(bad), bad[:3].tolist())
    if len(bad):
        e, a, f = bad[0]
        K = kw["k_nearest"]
        print(" dev row", dev[e, a, :4*K].reshape(K, 4)[:, :2].tolist())
        print(" ora row", ora[e, a, :4*K].reshape(K, 4)[:, :2].tolist())
    ws.close()
