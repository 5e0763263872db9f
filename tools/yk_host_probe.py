import sys, time; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1707_07598_b200 as gp
from paper_1707_07598_b200.models import table3_problem
from paper_1707_07598_b200.table3 import apply_Yk_dev, _csr_host
mesh, part, survey, m = table3_problem()
b = gp.BasisBuilder(part).assemble(gp.assemble_operator(mesh, torch.from_numpy(m).cuda()))
v = torch.from_numpy(np.random.default_rng(0).standard_normal(b.engine.k)).cuda()
md = torch.from_numpy(m).cuda()
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ip, ix, dv, shape = apply_Yk_dev(b, v, md); torch.cuda.synchronize(); t1 = time.perf_counter()
    a = ip.cpu().numpy(); t2 = time.perf_counter()
    c = ix.cpu().numpy(); t3 = time.perf_counter()
    d = dv.cpu().numpy(); t4 = time.perf_counter()
    import scipy.sparse as sp
    M = sp.csr_matrix((d, c, a.astype(np.int32)), shape=shape); t5 = time.perf_counter()
    print(f"dev {1e3*(t1-t0):.1f} ms, indptr {1e3*(t2-t1):.1f}, indices {1e3*(t3-t2):.1f}, data {1e3*(t4-t3):.1f}, csr {1e3*(t5-t4):.1f}")
    del a, c, d, M
    # pinned + async path
    t0 = time.perf_counter()
    hi = torch.empty(ix.shape, dtype=ix.dtype, pin_memory=True); hd = torch.empty(dv.shape, dtype=dv.dtype, pin_memory=True)
    t1 = time.perf_counter()
    hi.copy_(ix, non_blocking=True); hd.copy_(dv, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"  pinned alloc {1e3*(t1-t0):.1f} ms, copy {1e3*(t2-t1):.1f} ms")
    del hi, hd
