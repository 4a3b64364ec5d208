"""Envelope sweep (development tool, GPU box): every (nx, nu) near the
supported limit either solves within the parity bars or is rejected up front
with ValueError (CYQ_INVALID_ARG) -- never a CUDA error."""
import sys

sys.path.insert(0, "tests"); sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
from test_gpu_shapes import _problem  # noqa: E402
from pyoracle import Oracle  # noqa: E402
from paper_2512_09058_b200 import kkt  # noqa: E402
from paper_2512_09058_b200.ocp import EqRhsBatch, kkt_residual, rel_error  # noqa: E402

o = Oracle()
ok = rej = bad = 0
for nx in range(56, 92, 1):
    for nu in [1, 2, 3, 5, 8, 13, 16, 24, 40]:
        for P in [1, 16]:
            p = _problem(9, nx, nu, P, 1)
            try:
                s = kkt.solve_problem(p, kkt.FactorOptions(P=P))
            except ValueError:
                rej += 1
                continue
            except Exception as ex:
                bad += 1
                print(nx, nu, P, "EXC", repr(ex)[:160], flush=True)
                continue
            ref, rc, _ = o.solve_problem(p, P)
            e = rel_error(s, ref).max()
            r = kkt_residual(p, EqRhsBatch.of_problem(p), s).max()
            if e <= 1e-9 and r <= 1e-10:
                ok += 1
            else:
                bad += 1
                print(nx, nu, P, "err %.2e res %.2e" % (e, r), flush=True)
print(f"ok {ok} rejected {rej} bad {bad}")
