"""BASELINE config 2 on the GPU: bi-Maxwellian temperature isotropisation of one
cell of 1e5 electrons over 500 chained steps of the CUDA operator, against the
NRL Plasma Formulary law (the external closed form the oracle is pinned to,
tests/test_oracle_physics.py): the initial rate at dt/10 within 5% (as the
oracle's pin); at the nominal dt over 500 steps the energy 2 T_perp + T_par is
conserved to 1e-12, the log-decay of T_perp - T_par after ~2 e-folds is within
[0.75, 1.05] of the NRL ODE (TA's finite-dt sampler relaxes slower, DESIGN R5,
and the distribution leaves the bi-Maxwellian form the NRL law assumes), and
the anisotropy reaches the noise floor.  TA77 and the Nanbu variant (R20)."""
import numpy as np
import pytest

import workloads as W
from test_oracle_physics import nrl_rhs  # noqa: E402  (tests/ is on sys.path under pytest)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2508_06771_b200 as cc  # noqa: E402

DEV = torch.device("cuda:0")


def rk4(y, n, lnL, dt):
    k1 = nrl_rhs(*y, n, lnL)
    k2 = nrl_rhs(*(y + dt / 2 * k1), n, lnL)
    k3 = nrl_rhs(*(y + dt / 2 * k2), n, lnL)
    k4 = nrl_rhs(*(y + dt * k3), n, lnL)
    return y + dt / 6 * (k1 + 2 * k2 + 2 * k3 + k4)


def run_chain(w, flags, steps, dt, seed=None):
    p = w.params()
    p["dt"] = dt
    if seed is not None:
        p["seed"] = seed
    v, cell = torch.from_numpy(w.v).to(DEV), torch.from_numpy(w.cell).to(DEV)
    col = cc.Collider(w.n, 1, DEV, **{k: p[k] for k in ("dt", "weight", "cell_volume", "ln_lambda", "seed")})
    hist = [cc.cc_p2c_moments(cc.cc_p2c(v, cell, 1), weight=w.weight, cell_volume=w.cell_volume)[0].cpu().numpy()]
    for s in range(steps):
        out = col.step(v, cell, step=s, flags=flags)
        hist.append(out.moments[0].cpu().numpy())       # moments after step s
        v, cell = out.v_out, out.cell_out
    h = np.array(hist)
    return 0.5 * (h[:, 4] + h[:, 5]), h[:, 6]


def nrl_traj(tperp0, tpar0, n_e, lnL, dt, steps):
    y = np.array([tperp0, tpar0])
    ref = [y]
    for _ in range(steps):
        y = rk4(y, n_e, lnL, dt)
        ref.append(y)
    return np.array(ref)


@pytest.mark.parametrize("flags", [0, cc._lib.CC_NANBU])
@pytest.mark.parametrize("Tperp,Tpar", [(2.5, 1.0), (1.0, 2.5)])
def test_c2_isotropisation_matches_nrl(flags, Tperp, Tpar):
    w = W.c2(T_perp=Tperp, T_par=Tpar)
    n_e = w.n * w.weight / w.cell_volume
    # (1) the rate: at dt/10 (where TA's finite-dt sampler has converged to the Fokker-Planck
    #     limit, DESIGN R5) over the first 20 steps, while the distribution is still bi-Maxwellian.
    #     One chain's ratio scatters by ~5-6% (1e5 samples, 2% relaxation; measured with the oracle
    #     over 16 seeds: TA R1b 0.983, TA R1 0.962, Nanbu R1b 0.967, Nanbu R1 0.988, sd 0.04-0.06),
    #     so the rate is the mean over 16 collision seeds (sigma ~1.4%)
    ratios = []
    for seed in range(42, 58):
        tperp, tpar = run_chain(w, flags, 20, w.dt / 10, seed=seed)
        ref = nrl_traj(tperp[0], tpar[0], n_e, w.ln_lambda, w.dt / 10, 20)
        ratios.append(((tperp[-1] - tpar[-1]) - (tperp[0] - tpar[0])) /
                      ((ref[-1, 0] - ref[-1, 1]) - (ref[0, 0] - ref[0, 1])))
    ratio = float(np.mean(ratios))
    assert abs(ratio - 1.0) < 0.05, ratios
    # (2) config 2 as stated: 500 chained steps at the nominal dt — energy 2 T_perp + T_par
    #     conserved, the anisotropy decays at the NRL rate within the finite-dt and
    #     non-bi-Maxwellian margin, and reaches the noise floor
    tperp, tpar = run_chain(w, flags, 500, w.dt)
    e = 2 * tperp + tpar
    assert np.max(np.abs(e - e[0])) <= 1e-12 * e[0]
    ref = nrl_traj(tperp[0], tpar[0], n_e, w.ln_lambda, w.dt, 500)
    d_mc, d_ref = tperp - tpar, ref[:, 0] - ref[:, 1]
    k = 200                                   # ~2 e-folds of the anisotropy
    ratio = np.log(d_mc[k] / d_mc[0]) / np.log(d_ref[k] / d_ref[0])
    assert 0.75 < ratio < 1.05, ratio
    sigma = 2.0 * np.sqrt(2.0 / w.n)          # noise of a temperature estimate from 1e5 samples
    assert abs(d_mc[500]) < 0.02 * abs(d_mc[0]) + 4 * sigma
