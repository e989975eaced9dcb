"""Emulate the fp32 traversal arithmetic in numpy to size the guard.

For SIC decisions of sampled paths: index-domain centre error |a32 - a64|,
for (a) the shifted level-index form and (b) the symmetric odd-integer form,
with the rotation z in fp32 or fp64.  FMA is emulated as RN32(a*b + c)
evaluated in float64 (exact product)."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from oracle import mpnl_oracle as orc
from paper_2409_14355_b200.workloads import generate, CONFIGS
from paper_2409_14355_b200.core import constellation_for

f32 = np.float32
def fma(a, b, c):
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(f32)

def run(name, n_rb=2, paths=64, seed=3):
    cfg = CONFIGS[name]; d = generate(name, n_rb=n_rb, seed=seed)
    L = int(round(cfg.order ** 0.5)); nrm = np.sqrt(2 * (L * L - 1) / 3)
    plan = orc.plan_channels(d["h"], d["nv"][0], cfg.n_paths, cfg.order)
    rng = np.random.default_rng(1)
    errs = {"shift32": [], "sym32": [], "sym64z": []}
    mags = []
    for c in range(n_rb):
        R = plan.r[c]; QH = plan.qh[c]; N = cfg.n
        for v in range(0, d["y"].shape[1], 4):
            y = d["y"][c, v].astype(np.complex128)
            z64 = QH @ y
            y32 = d["y"][c, v]
            qh32 = QH.astype(np.complex64)
            # fp32 rotation with FMA order re: +qr*yr -qi*yi ; im: +qr*yi + qi*yr
            zr = np.zeros(N, f32); zi = np.zeros(N, f32)
            for m in range(cfg.m):
                qr, qi = qh32[:, m].real, qh32[:, m].imag
                yr, yi = np.full(N, y32[m].real, f32), np.full(N, y32[m].imag, f32)
                zr = fma(qr, yr, zr); zr = fma(-qi, yi, zr)
                zi = fma(qr, yi, zi); zi = fma(qi, yr, zi)
            # random symbol paths: decided symbols random (worst-ish) and also true-like
            for trial in range(paths):
                jr = rng.integers(0, L, N) * 2 - (L - 1)   # odd ints
                ji = rng.integers(0, L, N) * 2 - (L - 1)
                s = -(jr + 1j * ji) / nrm                   # symbol value
                for mode in ("shift32", "sym32", "sym64z"):
                    if mode == "shift32":
                        sc = (2 / nrm)
                        shift = (L - 1) / nrm * (1 + 1j) * np.array([R[k, k:].sum() for k in range(N)])
                        ar = (zr - f32(shift.real)).astype(f32); ai = (zi - f32(shift.imag)).astype(f32)
                        # level index i = (L-1 - j)/2 ... here s = (L-1-2i)/norm => i = (j+L-1)/2
                        ir = (jr + L - 1) // 2; ii = (ji + L - 1) // 2
                        coef = lambda k, p: (sc * R[k, p]).astype(np.complex64)
                        mult_r, mult_i = ir, ii
                    else:
                        if mode == "sym64z":
                            ar = z64.real.astype(f32); ai = z64.imag.astype(f32)
                        else:
                            ar, ai = zr.copy(), zi.copy()
                        coef = lambda k, p: (R[k, p] / nrm).astype(np.complex64)
                        mult_r, mult_i = jr, ji
                    ar = ar.copy(); ai = ai.copy()
                    for pos in range(N - 1, 0, -1):
                        cf = np.array([coef(k, pos) for k in range(pos)])
                        rr, ri = cf.real.astype(f32), cf.imag.astype(f32)
                        fr, fi = f32(mult_r[pos]), f32(mult_i[pos])
                        ar[:pos] = fma(rr, np.full(pos, fr), ar[:pos]); ar[:pos] = fma(-ri, np.full(pos, fi), ar[:pos])
                        ai[:pos] = fma(rr, np.full(pos, fi), ai[:pos]); ai[:pos] = fma(ri, np.full(pos, fr), ai[:pos])
                    # exact fp64 acc_k = z_k - sum_{j>k} r_kj s_j   (unshifted)
                    exact = np.array([z64[k] - R[k, k + 1:] @ s[k + 1:] for k in range(N)])
                    rkk = np.real(np.diag(R))
                    if mode == "shift32":
                        got = (ar.astype(np.float64) + 1j * ai) + (L - 1) / nrm * (1 + 1j) * rkk
                    else:
                        got = ar.astype(np.float64) + 1j * ai
                    # index-domain error: a = u*norm/(2 r)
                    err = np.abs(got - exact) * nrm / (2 * rkk)
                    errs[mode].append(np.maximum(err.real, err.imag) if np.iscomplexobj(err) else err)
            mags.append(np.abs(z64))
    for k, v in errs.items():
        a = np.concatenate(v)
        print(f"{name} {k:8s} median {np.median(a):.2e}  p99 {np.percentile(a,99):.2e}  max {a.max():.2e}")

for name in sys.argv[1:] or ["C2", "C4", "C5P64"]:
    run(name, n_rb=1, paths=16)
