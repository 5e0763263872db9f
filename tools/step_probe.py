"""Per-step device/host timing probe of the bench step (debug helper)."""
import gc, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_1707_07598_b200 as gp
from paper_1707_07598_b200.forward import forward_reduced_dev, sensitivity_adaptive
from paper_1707_07598_b200.models import config_problem

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mesh, part, survey, m = config_problem(cfg)
builder = gp.BasisBuilder(part)
m_dev = torch.from_numpy(m).cuda()
dobs = None


def step(check=True):
    op = gp.assemble_operator(mesh, m_dev)
    basis = builder.assemble(op)
    D, st = forward_reduced_dev(op, survey, basis, defer_check=True)
    st.deferred = True
    g = sensitivity_adaptive(st, survey).rapply_dev(D)
    if check:
        st.check()
    return g


step()
gc.collect()
gc.freeze()
for it in range(40):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    a.record()
    step(check=False)
    b.record()
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    h2 = time.perf_counter()
    ms = torch.cuda.memory_stats()
    print(f"step {it:2d} device {a.elapsed_time(b):7.3f} ms  host enqueue {1e3*(h1-h0):7.3f} ms  wall {1e3*(h2-h0):7.3f} ms"
          f"  alloc {torch.cuda.memory_allocated()/2**30:6.2f} GiB reserved {torch.cuda.memory_reserved()/2**30:6.2f}"
          f" mallocs {ms.get('num_device_alloc', -1)} frees {ms.get('num_device_free', -1)} gc {gc.get_count()}")
# back-to-back without sync
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    step(check=False)
b.record()
torch.cuda.synchronize()
print("back-to-back (no check)", a.elapsed_time(b) / 20)
a.record()
for _ in range(20):
    step(check=True)
b.record()
torch.cuda.synchronize()
print("back-to-back (check)", a.elapsed_time(b) / 20)
