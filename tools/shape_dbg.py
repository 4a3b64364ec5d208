"""Shape sweep against the C oracle (development tool, run on the GPU box):
python tools/shape_dbg.py -> one line per failing (N, nx, nu, P, batch) and a summary."""
import itertools
import sys

sys.path.insert(0, "tests"); sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
from test_gpu_shapes import _problem  # noqa: E402
from pyoracle import Oracle  # noqa: E402
from paper_2512_09058_b200 import kkt  # noqa: E402
from paper_2512_09058_b200.ocp import EqRhsBatch, kkt_residual, rel_error  # noqa: E402

o = Oracle()
NX = [1, 2, 3, 5, 8, 9, 12, 16, 17, 20, 24, 31, 32, 33, 40, 47, 48, 56, 64, 65, 72, 80, 96]
NU = [1, 4, 5, 8, 10, 16, 24, 32, 33, 48]
cases = [(11, nx, nu, 4, 2) for nx, nu in itertools.product(NX, NU)]
cases += [(N, nx, nu, P, b) for (N, P, b) in [(3, 8, 1), (33, 16, 3), (64, 2, 1), (1, 1, 1)]
          for nx, nu in [(10, 5), (20, 10), (12, 4), (16, 8), (64, 32), (7, 3), (40, 24)]]
bad = 0
for (N, nx, nu, P, b) in cases:
    p = _problem(N, nx, nu, P, b)
    ref, rc, _ = o.solve_problem(p, P)
    try:
        s = kkt.solve_problem(p, kkt.FactorOptions(P=P))
        e = rel_error(s, ref).max()
        r = kkt_residual(p, EqRhsBatch.of_problem(p), s).max()
        rr = kkt_residual(p, EqRhsBatch.of_problem(p), ref).max()
        if not (e <= 1e-9 and r <= 1e-10):
            bad += 1
            print(N, nx, nu, P, b, "err %.2e res %.2e (oracle res %.2e)" % (e, r, rr), flush=True)
    except Exception as ex:
        bad += 1
        print(N, nx, nu, P, b, "EXC", repr(ex)[:200], flush=True)
print(f"{len(cases)} cases, {bad} failing")
