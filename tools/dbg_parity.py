import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2603_08713_b200 as M
from oracle import mxq_oracle as O
from test_gpu_bench_parity import bench_inputs, oracle_view, M_TOK
dev = torch.device("cuda", 0)
va, vw = sys.argv[1], sys.argv[2]
n, k = int(sys.argv[3]), int(sys.argv[4])
a, w = bench_inputs(dev, k, n, 77)
wq = M.quantize_tensor(w, M.SchemeConfig(M.Variant(vw)))
aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant(va)))
rows = np.r_[0:128, M_TOK - 128:M_TOK]
c = M.matmul_quantized(aq, wq).cpu().numpy()[rows].astype(np.float64)
da_o = O.dequantize(oracle_view(aq, rows)).astype(np.float64)
db_o = O.dequantize(oracle_view(wq)).astype(np.float64)
da_g = M.dequantize_tensor(aq).cpu().numpy()[rows].astype(np.float64)
db_g = M.dequantize_tensor(wq).cpu().numpy().astype(np.float64)
print("dequant equal A", np.array_equal(da_o, da_g), "B", np.array_equal(db_o, db_g))
want = da_o @ db_o.T
err = np.abs(c - want)
print("rel fro", np.linalg.norm(c - want) / np.linalg.norm(want))
r, col = np.unravel_index(np.argmax(err), err.shape)
print("worst", rows[r], col, c[r, col], want[r, col])
rowerr = np.linalg.norm(c - want, axis=1) / np.linalg.norm(want, axis=1)
print("rows with rel>1e-4:", [(int(rows[i]), float(rowerr[i])) for i in np.argsort(-rowerr)[:10]])
colerr = np.linalg.norm(c - want, axis=0) / np.linalg.norm(want, axis=0)
bad = np.where(colerr > 1e-4)[0]
print("n bad cols", len(bad), bad[:20], bad[-20:] if len(bad) else None)
ex = M.matmul_quantized(aq, wq, exact=True).cpu().numpy()[rows].astype(np.float64)
print("exact rel fro", np.linalg.norm(ex - want) / np.linalg.norm(want))
