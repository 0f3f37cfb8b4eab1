"""How coarse can the filter's per-target summary be? For C2 layer-2 PAIRs of a
few rounds: fraction of PAIRs settled irrelevant (u < alpha at every position,
max aggregation) by group tests min_{i in g} alpha_i > max_{i in g} u_i for
group sizes 1 (exact), 2, 4, 8, 16, 32."""
import json, os, sys
import numpy as np
ROOT = '/root/repo'
sys.path.insert(0, ROOT)
import bench
import paper_2309_11071_b200 as sg
from tools import configs as CF
gen, src, dst, feats, desc, man = bench.product_inputs('c2')
n = CF.CONFIGS['c2']['nodes']
g = sg.Graph.from_edges(n, src, dst)
e = sg.Engine.create_from_array(g, sg.Model.load(desc, man), feats)
# out-lists of the initial graph (CSR from the arrays)
order = np.argsort(src, kind='stable'); s_sorted = src[order]; d_sorted = dst[order]
starts = np.searchsorted(s_sorted, np.arange(n + 1))
res = {G: [0, 0] for G in (1, 32, 64, 128, 256)}
d2 = 256
for rnd, (ops, ss, dd) in enumerate(CF.batches('c2', gen, src, dst, 4)):
    old = e.read_table(2, 0)
    e.apply_update(ops, ss, dd)
    new = e.read_table(2, 0)
    alpha = e.read_table(2, 1)   # after the round; PAIR relevance is judged against alpha_prev but this is close
    base = alpha.min(axis=0); rng = np.maximum(alpha.max(axis=0) - base, 1e-30)
    alpha_n = (alpha - base) / rng   # per-column normalised (what the 16-bit codes quantise)
    dirty = e.dirty_nodes(1)
    for j in dirty:
        u = (np.maximum(old[j], new[j]) - base) / rng
        tg = d_sorted[starts[j]:starts[j + 1]]
        if len(tg) == 0: continue
        A = alpha_n[tg]         # (T, 256)
        for G in res:
            amin = A.reshape(len(tg), d2 // G, G).min(axis=2)
            umax = u.reshape(d2 // G, G).max(axis=1)
            settled = (amin > umax[None, :]).all(axis=1)
            res[G][0] += int(settled.sum()); res[G][1] += len(tg)
print(json.dumps({G: round(a / max(b, 1), 4) for G, (a, b) in res.items()}), res[1][1])
