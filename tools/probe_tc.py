import numpy as np, torch
from paper_2605_17913_b200 import capi
dev = torch.device("cuda:0")
def run(G, om, n):
    p = G.shape[0]
    Q = np.zeros((n, n), np.float32)
    tG, tom, tQ = (torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev) for a in (G, om, Q))
    tH = torch.zeros((n, n), device=dev)
    capi.qp_debug_tc_syrk(tG.data_ptr(), tom.data_ptr(), tQ.data_ptr(), n, p, tH.data_ptr())
    torch.cuda.synchronize()
    return tH.cpu().numpy()
n = 128
for (k, a, b) in [(0, 0, 0), (0, 1, 1), (0, 4, 4), (0, 5, 9), (1, 0, 0), (3, 2, 2), (8, 0, 0), (9, 3, 7), (0, 0, 64), (17, 33, 100)]:
    G = np.zeros((32, n), np.float32); G[k, a] = 1; G[k, b] += 2
    H = run(G, np.ones(32, np.float32), n)
    nz = np.argwhere(H != 0)
    print(f"k={k} a={a} b={b}:", [(int(i), int(j), float(H[i, j])) for i, j in nz[:8]], len(nz))
