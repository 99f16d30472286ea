"""Does running the CholQR2's memory-bound passes (SK -> canonical layout,
X R^-1) concurrently with its tensor-bound Grams pay?  Times, at config 4's
size: each kernel alone, pairs on two streams, and a row-chunk pipeline
X R^-1 (chunk k) -> Gram (chunk k) on a second stream.
Usage: overlap_probe.py [n] [r] [chunks]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(n, r, chunks):
    from paper_2601_18705_b200 import _lib
    from paper_2601_18705_b200.mesh import build_grid, cellops_struct

    lib = _lib.load()
    grid = build_grid(n, n, (0.0, 0.0, 1.0, 1.0))
    co = cellops_struct(grid)
    N = grid.n_dofs
    vl = int(lib.dlrsn_sk_vec_len(n, n))
    dev = torch.device("cuda")
    psi_sk = torch.rand(r * vl, dtype=torch.float64, device=dev)
    psi = torch.rand(N, r, dtype=torch.float64, device=dev)
    X1 = torch.empty(N, r, dtype=torch.float64, device=dev)
    other = torch.rand(N, r, dtype=torch.float64, device=dev)
    quads = (torch.arange(r, device=dev, dtype=torch.int32) % 4).contiguous()
    Rinv = torch.triu(torch.rand(r, r, dtype=torch.float64, device=dev)).contiguous()
    G = torch.empty(chunks + 1, r, r, dtype=torch.float64, device=dev)
    part = torch.empty(int(lib.dlrsn_partials_len(grid.n_cells, r, r, 0)), dtype=torch.float64, device=dev)
    part2 = torch.empty_like(part)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    P = lambda t: _lib.ptr(t)
    H = lambda s: ctypes.c_void_p(s.cuda_stream)

    def to_canon(s):
        _lib.call("dlrsn_sk_to_canonical", ctypes.byref(co), r, P(quads), P(psi_sk), P(psi), r, H(s))

    def gram(src, s, out=None, pt=None):
        _lib.call("dlrsn_mgram", ctypes.byref(co), r, r, P(src), r, P(src), r, None,
                  P(G[0] if out is None else out), P(part if pt is None else pt), H(s))

    def rmix(s):
        _lib.call("dlrsn_rowmix_upper", N, r, P(psi), r, P(Rinv), r, P(X1), r, H(s))

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    cur = torch.cuda.current_stream()

    def pair(a, b):
        def run():
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            a(s1)
            b(s2)
            cur.wait_stream(s1)
            cur.wait_stream(s2)
        return run

    print(f"n={n} r={r}: sk_to_canonical {timed(lambda: to_canon(cur)):.3f} ms, "
          f"mgram {timed(lambda: gram(other, cur)):.3f} ms, rowmix_upper {timed(lambda: rmix(cur)):.3f} ms")
    print(f"  sk_to_canonical || mgram(other): {timed(pair(to_canon, lambda s: gram(other, s))):.3f} ms")
    print(f"  rowmix_upper    || mgram(other): {timed(pair(rmix, lambda s: gram(other, s))):.3f} ms")
    print(f"  serial rowmix_upper -> mgram(X1): {timed(lambda: (rmix(cur), gram(X1, cur))):.3f} ms")

    # row-chunk pipeline: X1 rows of chunk k on s1, their Gram on s2
    rows = n // chunks
    sub = build_grid(n, rows, (0.0, 0.0, 1.0, rows / n))
    cs = cellops_struct(sub)
    evs = [torch.cuda.Event() for _ in range(chunks)]

    def pipeline():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        for k in range(chunks):
            o = 4 * n * rows * k
            _lib.call("dlrsn_rowmix_upper", 4 * n * rows, r, P(psi[o:]), r, P(Rinv), r, P(X1[o:]), r, H(s1))
            evs[k].record(s1)
            s2.wait_event(evs[k])
            _lib.call("dlrsn_mgram", ctypes.byref(cs), r, r, P(X1[o:]), r, P(X1[o:]), r, None,
                      P(G[k + 1]), P(part2), H(s2))
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    print(f"  pipeline of {chunks} row chunks (rowmix_upper on s1 -> mgram on s2): {timed(pipeline):.3f} ms")
    gram(X1, cur)
    torch.cuda.synchronize()
    err = (G[1:].sum(0) - G[0]).abs().max().item() / G[0].abs().max().item()
    print(f"  chunked Gram vs whole: rel diff {err:.2e}")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(int(a[0]) if a else 1024, int(a[1]) if len(a) > 1 else 64, int(a[2]) if len(a) > 2 else 16)
