"""Host-side overhead probe of the public fmm_evaluate call (pinned buffers)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1205_4611_b200 as F
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
rng = np.random.default_rng(1)
h_pos = torch.empty(n, dtype=torch.complex128, pin_memory=True).numpy()
h_pos[:] = rng.uniform(size=n) + 1j * rng.uniform(size=n)
h_g = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
h_g[:] = rng.uniform(-1, 1, n)
h_out = torch.empty(n, dtype=torch.complex128, pin_memory=True).numpy()
ps = F.ParticleSet(h_pos, h_g)
cfg = F.TreeConfig(35, 0.5, 20)   # n_desired_per_box, theta, p_terms (C2)
for _ in range(3):
    F.fmm_evaluate(ps, cfg, out=h_out)
ts, dev, tot = [], [], []
for _ in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, r = F.fmm_evaluate(ps, cfg, out=h_out)
    ts.append(time.perf_counter() - t0)
    dev.append(r.device_seconds)
print(f"wall {np.mean(ts)*1e3:.3f} ms  device {np.mean(dev)*1e3:.3f} ms  "
      f"c_total {r.total_seconds*1e3:.3f}")
# raw copy speeds
d = torch.empty(n, dtype=torch.complex128, device='cuda')
torch.cuda.synchronize()
t0 = time.perf_counter(); d.copy_(torch.from_numpy(h_pos), non_blocking=True); torch.cuda.synchronize()
t1 = time.perf_counter(); torch.from_numpy(h_out).copy_(d, non_blocking=True); torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"H2D 16MB {1e3*(t1-t0):.3f} ms  D2H 16MB {1e3*(t2-t1):.3f} ms")
