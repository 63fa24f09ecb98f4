import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_08713_b200 as M
dev = torch.device("cuda", 0)
def run(m, n, k, seed=1):
    g = torch.Generator(device=dev).manual_seed(seed)
    a = torch.randn(m, k, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, device=dev, generator=g) * 0.02).to(torch.bfloat16)
    wq = M.quantize_tensor(w, M.SchemeConfig(M.Variant.MBS_D))
    aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant.MBS_S))
    ex = M.matmul_quantized(aq, wq, exact=True).double()
    c = M.matmul_quantized(aq, wq).double()
    err = (c - ex).abs() > 1e-4 * ex.abs().max()
    nb = int(err.sum())
    out = f"{m}x{n}x{k}: relfro {float((c-ex).norm()/ex.norm()):.2e} bad {nb}"
    if nb:
        r, cc = err.nonzero(as_tuple=True)
        q = (r % 128) // 32; grp = (cc % 192) // 48; cl = cc % 48
        tab = torch.zeros(4, 4, dtype=torch.int64, device=dev)
        tab.index_put_((q, grp), torch.ones_like(q), accumulate=True)
        out += f"\n   quad x grp counts {tab.tolist()}  col-in-grp hist {torch.bincount(cl, minlength=48).tolist()}"
        tiles = (r // 128) * ((n + 191) // 192) + cc // 192
        out += f"\n   distinct tiles {len(torch.unique(tiles))} of {((m+127)//128)*((n+191)//192)}"
    print(out, flush=True)
    return aq, wq, c, ex, err
for shp in [(1024, 1536, 4096), (4096, 6144, 1024), (4096, 6144, 2048), (2048, 3072, 4096), (4096, 6144, 4096)]:
    run(*shp)
