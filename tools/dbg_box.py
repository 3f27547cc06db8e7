import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2508_10076_b200 import tk
from workloads import configs as W
from oracle import layout as OL, blocksparse as BS, contract as OC
for d in (96, 128):
    V = W.cfg4_leg(d)
    cod, dom = [V, V], [V, V]
    for p, q in (([0, 2], [1, 3]), ([2, 0], [1, 3]), ([0, 3], [2, 1]), ([0, 1, 3], [2])):
        lt = OL.homspace_layout("U1", cod, dom)
        x = np.random.default_rng(0).standard_normal(lt.nelems)
        c2, d2 = OC.permuted_spaces(cod, dom, p, q)
        ls = OL.homspace_layout("U1", c2, d2)
        A = tk.tensor_from_spec({"cod": cod, "dom": dom}); C = tk.tensor_from_spec({"cod": c2, "dom": d2})
        a = torch.from_numpy(x).cuda(); c = torch.full((ls.nelems,), float("nan"), dtype=torch.float64, device="cuda")
        tk.tk_permute(A, a, p, q, C, c)
        torch.cuda.synchronize()
        got = c.cpu().numpy()
        # reference via subblocks: every A subblock, transposed, lands in its C subblock
        xa = BS.to_blocks(lt, x)
        gc = BS.to_blocks(ls, got)
        order = list(p) + list(q)
        err = 0.0; nbad = 0
        for k, v in xa.items():
            kc = tuple(k[i] for i in order)
            # dual flips: U1 label sign flips when a leg crosses cod/dom
            kk = []
            for pos, i in enumerate(order):
                was_cod, now_cod = i < 2, pos < len(p)
                kk.append(k[i] if was_cod == now_cod else (-k[i][0],))
            r = np.transpose(v, order)
            g = gc[tuple(kk)]
            e = np.abs(g - r).max()
            if e > 0: nbad += 1
            err = max(err, e)
        print(d, p, q, "maxerr", err, "bad subblocks", nbad, "of", len(xa))
