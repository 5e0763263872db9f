"""Find host synchronisations and GPU idle time in the device-resident step."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_1707_07598_b200 as gp
from paper_1707_07598_b200.forward import forward_reduced_dev, sensitivity_adaptive
from paper_1707_07598_b200.models import config_problem
mesh, part, survey, m = config_problem(4)
builder = gp.BasisBuilder(part)
m_dev = torch.from_numpy(m).cuda()
def step(defer=True):
    op = gp.assemble_operator(mesh, m_dev)
    basis = builder.assemble(op)
    D, st = forward_reduced_dev(op, survey, basis, defer_check=defer)
    st.deferred = True
    g = sensitivity_adaptive(st, survey).rapply_dev(D)
    st.check()
    return g
for _ in range(3): step()
torch.cuda.synchronize()
torch.cuda.set_sync_debug_mode("warn")
t = time.perf_counter(); step(); t_enq = time.perf_counter() - t
torch.cuda.set_sync_debug_mode(0)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); a.record(); step(); b.record(); torch.cuda.synchronize(); wall = time.perf_counter() - t0
print(f"enqueue-until-check {t_enq*1e3:.2f} ms, wall {wall*1e3:.2f} ms, events {a.elapsed_time(b):.2f} ms")
for n in (1, 5, 10):
    torch.cuda.synchronize()
    a.record()
    for _ in range(n): step()
    b.record(); torch.cuda.synchronize()
    print(f"{n} steps: {a.elapsed_time(b)/n:.2f} ms/step")
from paper_1707_07598_b200.engine import PhaseTimer
PhaseTimer.start(); step(); ph = PhaseTimer.stop()
print("phase sum", sum(ph.values()), ph)
print(torch.cuda.memory_stats()["num_alloc_retries"], torch.cuda.max_memory_allocated() / 1e9)
evs = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
evs[0].record()
for i in range(20):
    step(); evs[i + 1].record()
torch.cuda.synchronize()
print("per-step ms:", " ".join(f"{evs[i].elapsed_time(evs[i+1]):.2f}" for i in range(20)))
st0 = torch.cuda.memory_stats()
print({k: v for k, v in st0.items() if "num_device" in k or "alloc_retries" in k or "num_sync" in k})
import gc
def step_nocheck():
    op = gp.assemble_operator(mesh, m_dev)
    basis = builder.assemble(op)
    D, st = forward_reduced_dev(op, survey, basis, defer_check=True)
    st.deferred = True
    return sensitivity_adaptive(st, survey).rapply_dev(D)
torch.cuda.synchronize()
t = time.perf_counter(); step_nocheck(); th = time.perf_counter() - t; torch.cuda.synchronize()
print(f"pure host enqueue {th*1e3:.2f} ms")
for dis in (False, True):
    if dis: gc.collect(); gc.disable()
    torch.cuda.synchronize(); a.record()
    for _ in range(10): step()
    b.record(); torch.cuda.synchronize()
    print(f"gc disabled={dis}: 10 steps {a.elapsed_time(b)/10:.2f} ms/step, gc counts {gc.get_count()}")
gc.enable()
