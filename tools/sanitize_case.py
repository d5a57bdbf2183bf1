"""Small engine runs for compute-sanitizer (racecheck / synccheck / memcheck):
both summation modes, multi-RHS waves (one CTA per right-hand side) and the
single-RHS cluster path (the coarse march), the rolling-window ILUT streams,
the device ILUT and the V-cycle kernel.  Tiny shapes: the tools replay every
shared-memory access.   python tools/sanitize_case.py [window]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_05337_b200 as P  # noqa: E402

P.lib().phi_set_device(0)
for exact in (False, True):
    d = P.SpatialDiscretization.build(2, 3)
    s = P.MgritSolver(d, 16, m=4, cycle=P.CYCLE_TWO_LEVEL, source_param=0.0, init_kind=P.INIT_SIN, exact=exact)
    r = s.solve()
    print(f"mgrit exact={exact}: {r.iterations} iterations, {r.total_spatial_solves} solves", flush=True)
    h = P.PMultigridHierarchy(d, 1e-3, exact=exact)
    b = np.random.default_rng(0).standard_normal((3, d.n_free))
    h.vcycle(b, np.zeros_like(b))
    print(f"vcycle exact={exact} ok", flush=True)
if len(sys.argv) > 1 and sys.argv[1] == "window":
    # a shape whose ILUT vector does not fit in shared memory: rolling-window streams
    d = P.SpatialDiscretization.build(4, 7)
    st = P.ThetaStepper(d, 1.0, 1.6e-4, 1.0)
    u = np.random.default_rng(1).uniform(-1, 1, d.n_free)
    st.step(u)
    print("window-stream step ok", flush=True)
