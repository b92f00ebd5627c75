"""One dense-split GEMM (pack + gemm) per process: rel err of f16x2 / bf16x3
against float64, with the max |x| per row spanning several decades."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2306_15155_b200 import _native as nat
K, T, fmt, spread = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
f = nat.GC_HUB_F16X2 if fmt == "f16x2" else nat.GC_HUB_BF16X3
dt = torch.float16 if fmt == "f16x2" else torch.bfloat16
terms = 2 if fmt == "f16x2" else 3
rng = np.random.default_rng(K * 7 + T)
n, ncols = 777, 3000
a_hub = (rng.random((n, T)) < 0.3).astype(np.float32)
x = (rng.standard_normal((ncols, K)) * 10.0 ** rng.integers(-spread, spread + 1, (ncols, 1))).astype(np.float32)
hub_cols = np.sort(rng.choice(ncols, T, replace=False)).astype(np.int32)
d = rng.uniform(0.05, 1.0, ncols).astype(np.float32)
dr = rng.uniform(0.05, 1.0, n).astype(np.float32)
lib = nat.load(); dev = "cuda"
kp = lib.gc_hub_terms_rows(K)
bt = torch.empty(terms * kp * T, dtype=dt, device=dev)
sc = torch.zeros(2, dtype=torch.float32, device=dev)
xt, ht, dtt, drt = (torch.from_numpy(v).to(dev) for v in (x, hub_cols, d, dr))
at = torch.from_numpy(a_hub).to(dev).to(dt)
out = torch.full((n, K), float("nan"), device=dev)
st = torch.cuda.current_stream().cuda_stream
nat.check(lib.gc_hub_pack(xt.data_ptr(), K, K, ht.data_ptr(), T, dtt.data_ptr(), f, bt.data_ptr(), sc.data_ptr(), st), "pack")
nat.check(lib.gc_hub_gemm(at.data_ptr(), T, n, T, bt.data_ptr(), K, f, sc.data_ptr(), out.data_ptr(), K, drt.data_ptr(), 0, st), "gemm")
torch.cuda.synchronize()
xs = x.astype(np.float64)[hub_cols] * d.astype(np.float64)[hub_cols][:, None]
ref = dr.astype(np.float64)[:, None] * (a_hub.astype(np.float64) @ xs)
o = out.cpu().numpy()
err = np.abs(o - ref).max() / max(1.0, np.abs(ref).max())
# emulate: hi only / hi+lo in numpy
s_ = sc.cpu().numpy()
print(f"K={K} T={T} {fmt} spread={spread}: rel_err={err:.3e} amax_bits->{np.frombuffer(s_[:1].tobytes(), np.float32)[0]:.4g} inv_scale={s_[1]:.4g} max|xs|={np.abs(xs).max():.4g}")
if fmt == "f16x2":
    s = 1.0 / s_[1]
    y = (xs * s).astype(np.float32)
    hi = y.astype(np.float16).astype(np.float32)
    lo = (y - hi).astype(np.float16).astype(np.float32)
    b16 = bt.view(torch.float16).cpu().numpy().astype(np.float32).reshape(2, kp, T)
    print("  pack hi matches:", np.allclose(b16[0, :K, :], hi.T), " lo matches:", np.allclose(b16[1, :K, :], lo.T),
          " lo nonzero:", float(np.abs(b16[1]).max()))
    emu_hi = dr[:, None].astype(np.float64) * (a_hub.astype(np.float64) @ (hi.astype(np.float64) / s))
    print("  emulated hi-only err:", np.abs(emu_hi - ref).max() / max(1.0, np.abs(ref).max()))
