"""Exact line search of the QPALM inner loop:
qpalm::line_search_exact (line_search.cpp:112-206) over
LineSearchData::add_term (line_search.cpp:9-27).

CPU (pins the oracle): the C restatement (oracle/cyq_oracle.c) against the
reference's own line_search.cpp compiled into oracle/_ref, on the reference
test's closed forms and folding rules (test_line_search.cpp:35-92) and on
seeded random instances; GPU: cyq_line_search_batch against both, edge
cases, determinism, and the optimality property the reference test checks
(|psi'(tau)| small relative to the breakpoint scale, test_line_search.cpp:
139-162).
"""
import numpy as np
import pytest

from pyoracle import Oracle, RefOracle, ref_available

from paper_2512_09058_b200 import synth

INF = np.inf


def psi_prime(alpha, delta, eta, beta, tau):
    """The defining sum (line_search.hpp:19-21) with add_term's filters."""
    with np.errstate(divide="ignore", invalid="ignore"):
        t = alpha / delta
    keep = (delta != 0) & np.isfinite(t)
    d, a = delta[keep], alpha[keep]
    return eta * tau + beta + np.sum(d * np.maximum(d * tau - a, 0.0))


def scale_of(alpha, delta, eta):
    with np.errstate(divide="ignore", invalid="ignore"):
        t = alpha / delta
    keep = (delta != 0) & np.isfinite(t)
    w = delta[keep] * np.abs(delta[keep])
    return max(1.0, abs(eta)) + np.sum(np.abs(w) * np.maximum(1.0, np.abs(t[keep])))


# closed forms of test_line_search.cpp:35-74, as (alpha, delta, eta, beta, tau)
KATS = [
    (np.zeros(0), np.zeros(0), 2.0, -2.0, 1.0),                # no breakpoints
    (np.array([0.5]), np.array([1.0]), 1.0, -1.0, 0.75),       # one breakpoint t = 0.5, w = 1
    # folding: delta = 0 dropped, infinite alpha dropped, t = -0.5 (w > 0)
    # folded into eta / beta (eta 1 + 4, beta -5 + 2), t = -0.5 (w < 0) never active
    (np.array([1.0, INF, -1.0, 1.0]), np.array([0.0, 1.0, 2.0, -2.0]), 1.0, -5.0, 0.6),
]


@pytest.mark.parametrize("case", range(len(KATS)))
def test_oracle_closed_forms(case):
    alpha, delta, eta, beta, tau = KATS[case]
    got, rc = Oracle().line_search(alpha[None], delta[None], [eta], [beta])
    assert rc[0] == 0 and abs(got[0] - tau) <= 1e-15 * max(1.0, abs(tau))


def test_oracle_non_descent_and_flat():
    tau, rc = Oracle().line_search(np.zeros((2, 0)), np.zeros((2, 0)), [1.0, 1.0], [0.5, 0.0])
    assert list(rc) == [1, 0] and tau[1] == 0.0


@pytest.mark.skipif(not ref_available(), reason="reference build not available")
def test_oracle_matches_reference_build():
    alpha, delta, eta, beta = synth.line_search_data(40, 700, seed=3)
    alpha[5, :] = INF          # no breakpoints at all
    delta[6, :] = 0.0
    beta[7] = 0.3              # not a descent direction
    beta[8] = 0.0              # flat
    mine, rc_m = Oracle().line_search(alpha, delta, eta, beta)
    ref, rc_r, _ = RefOracle().line_search(alpha, delta, eta, beta)
    assert np.array_equal(rc_m, rc_r)
    ok = rc_r == 0
    assert np.all(np.abs(mine[ok] - ref[ok]) <= 1e-12 * np.maximum(1.0, np.abs(ref[ok])))
    for alpha_, delta_, eta_, beta_, tau_ in KATS:
        r, c, _ = RefOracle().line_search(alpha_[None], delta_[None], [eta_], [beta_])
        assert c[0] == 0 and abs(r[0] - tau_) <= 1e-15 * max(1.0, abs(tau_))


@pytest.mark.gpu
def test_gpu_line_search_matches_reference():
    import torch
    from paper_2512_09058_b200 import kkt

    alpha, delta, eta, beta = synth.line_search_data(96, 2 * 24 * 65, seed=11)
    alpha[3, :] = INF            # no breakpoints: tau = -beta / eta
    alpha[4, :50] = np.linspace(0.001, 0.05, 50) * delta[4, :50]  # a cluster of tiny breakpoints
    delta[5, :] = 0.0
    dev = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (alpha, delta, eta, beta)]
    tau = kkt.line_search_exact(*dev).cpu().numpy()
    ref, rc, _ = (RefOracle().line_search(alpha, delta, eta, beta) if ref_available()
                  else (*Oracle().line_search(alpha, delta, eta, beta), None))
    assert np.all(rc == 0)
    assert np.all(np.abs(tau - ref) <= 1e-12 * np.maximum(1.0, np.abs(ref)))
    for b in range(0, 96, 7):
        assert abs(psi_prime(alpha[b], delta[b], eta[b], beta[b], tau[b])) <= \
            1e-10 * scale_of(alpha[b], delta[b], eta[b])
    # deterministic: a second launch is bit-identical
    assert np.array_equal(tau, kkt.line_search_exact(*dev).cpu().numpy())


@pytest.mark.gpu
def test_gpu_line_search_edge_cases():
    import torch
    from paper_2512_09058_b200 import kkt

    # the closed forms, one instance each (padded with dropped terms)
    m = 4
    rows = []
    for alpha, delta, eta, beta, tau in KATS:
        a = np.full(m, INF)
        d = np.zeros(m)
        a[:len(alpha)], d[:len(delta)] = alpha, delta
        rows.append((a, d, eta, beta, tau))
    A = np.stack([r[0] for r in rows])
    D = np.stack([r[1] for r in rows])
    E = np.array([r[2] for r in rows])
    B = np.array([r[3] for r in rows])
    dev = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (A, D, E, B)]
    tau = kkt.line_search_exact(*dev).cpu().numpy()
    for (_, _, _, _, t), g in zip(rows, tau):
        assert abs(g - t) <= 1e-15 * max(1.0, abs(t))
    # non-descent raises (std::invalid_argument in the reference); flat -> 0
    E2 = torch.tensor([1.0, 1.0], dtype=torch.float64, device="cuda")
    B2 = torch.tensor([0.5, 0.0], dtype=torch.float64, device="cuda")
    Z = torch.zeros((2, 3), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        kkt.line_search_exact(Z, Z, E2, B2)
    t2, st = kkt.line_search_exact(Z, Z, E2, B2, raise_on_error=False)
    assert st[0] != 0 and st[1] == 0 and float(t2[1]) == 0.0


@pytest.mark.gpu
def test_gpu_line_search_root_beyond_last_breakpoint_and_below_first():
    import torch
    from paper_2512_09058_b200 import kkt

    # weak curvature: the root lies beyond every breakpoint / strong: below all
    rng = np.random.default_rng(4)
    m = 300
    delta = rng.uniform(0.5, 1.0, (2, m))
    alpha = rng.uniform(0.1, 1.0, (2, m)) * delta   # breakpoints in (0.1, 1)
    eta = np.array([1e-6, 1e6])
    beta = np.array([-1e3, -1.0])
    dev = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (alpha, delta, eta, beta)]
    tau = kkt.line_search_exact(*dev).cpu().numpy()
    ref, rc = Oracle().line_search(alpha, delta, eta, beta)
    assert np.all(rc == 0)
    assert tau[0] > 1.0 and tau[1] < 0.1
    assert np.all(np.abs(tau - ref) <= 1e-12 * np.maximum(1.0, np.abs(ref)))


@pytest.mark.gpu
def test_gpu_line_search_without_terms_and_large_batch():
    import torch
    from paper_2512_09058_b200 import kkt

    # m = 0: psi' is linear, tau = -beta / eta (line_search.cpp:140-146)
    E = torch.tensor([2.0, 4.0], dtype=torch.float64, device="cuda")
    B = torch.tensor([-2.0, -1.0], dtype=torch.float64, device="cuda")
    Z = torch.zeros((2, 0), dtype=torch.float64, device="cuda")
    tau = kkt.line_search_exact(Z, Z, E, B).cpu().numpy()
    assert np.allclose(tau, [1.0, 0.25], rtol=0, atol=1e-15)
    # a batch larger than the SM count, small m: every instance vs the oracle
    alpha, delta, eta, beta = synth.line_search_data(700, 37, seed=21)
    dev = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (alpha, delta, eta, beta)]
    got = kkt.line_search_exact(*dev).cpu().numpy()
    ref, rc = Oracle().line_search(alpha, delta, eta, beta)
    assert np.all(rc == 0)
    assert np.all(np.abs(got - ref) <= 1e-12 * np.maximum(1.0, np.abs(ref)))
