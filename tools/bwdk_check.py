"""Stress check of the C4 backward-kernel convolutions: integer inputs in {-1,0,1}
(exact in any summation order) at several batch sizes, repeated evaluations;
prints mismatch counts per run (a race shows up as run-to-run variation)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1812_03770_b200 import cg  # noqa: E402


def ref_bwdk(x, dy, ks, pad):
    n, h, w, ci = x.shape
    _, ho, wo, co = dy.shape
    p = (ks - 1) // 2 if pad else 0
    xp = np.zeros((n, ho + ks - 1, wo + ks - 1, ci))
    xp[:, p:p + h, p:p + w, :] = x
    out = np.zeros((ks, ks, ci, co))
    for kh in range(ks):
        for kw in range(ks):
            out[kh, kw] = np.einsum("nhwc,nhwo->co", xp[:, kh:kh + ho, kw:kw + wo, :], dy, optimize=True)
    return out


def main():
    geos = [((28, 28, 1), 6, 28, 1), ((14, 14, 6), 16, 10, 0)]
    for (h, w, ci), co, ho, pad in geos:
        for batch in [int(b) for b in (sys.argv[1:] or ["300", "2400", "8192"])]:
            rng = np.random.default_rng(batch)
            x = rng.integers(-1, 2, (batch, h, w, ci)).astype(np.float32)
            dy = rng.integers(-1, 2, (batch, ho, ho, co)).astype(np.float32)
            ref = ref_bwdk(x.astype(np.float64), dy.astype(np.float64), 5, pad)
            g = cg.Graph(0)
            vx, vd = g.var(x.shape), g.var(dy.shape)
            o = g.add_node("CONV2D_BWD_KERNEL", [vx, vd], sh=1, sw=1, pad=pad, kh=5, kw=5)
            g.plan_memory([o])
            g.assign(vx, x)
            g.assign(vd, dy)
            res = []
            for _ in range(4):
                g.eval([o])
                got = g.read(o).astype(np.float64)
                bad = np.argwhere(got != ref)
                res.append((len(bad), float(np.abs(got - ref).max())))
            print(f"ci={ci} co={co} batch={batch}: mismatches per run {res}", flush=True)
            if res[0][0]:
                got = g.read(o).astype(np.float64)
                bad = np.argwhere(got != ref)
                print("  first bad (kh,kw,ci,co):", bad[:8].tolist(), flush=True)
                d = (got - ref).reshape(-1, got.shape[-1])
                print("  bad per co:", (d != 0).sum(0).tolist())
                print("  bad rows (m):", sorted(set(np.argwhere(d != 0)[:, 0].tolist()))[:40])
                print("  diff row 0:", d[0].tolist())


if __name__ == "__main__":
    main()
