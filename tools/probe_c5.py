"""Config-5 kernel microbenchmark preview: SpMM GB/s (A read once) and V-cycle."""
import sys
sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for p in (2, 3, 4, 5):
    d = P.SpatialDiscretization.build(p, k)
    h = P.PMultigridHierarchy(d, 1e-4)
    n = d.n_free
    nnz = (int(round(n ** 0.5)) * (2 * p + 1) - p * (p + 1)) ** 2
    for b in (1, 16, 64):
        ms = h.time_kernel(0, b, reps=5)
        by = 8 * nnz + b * 16 * n
        print(f"p={p} B={b:2d}: spmm {ms * 1e3:8.1f} us  {by / ms / 1e6:7.0f} GB/s (alg {by / 1e6:.1f} MB)", flush=True)
