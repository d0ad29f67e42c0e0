"""Shared test helpers: seeded synthetic inputs and tolerances."""

import numpy as np

from oracle import lbscan_oracle as O

TOL_F32 = 1e-5     # north star: fp32 path, max_rel_err (core.py:149-156)
TOL_BF16 = 2e-2    # bf16 inputs with fp32 state
TOL_GRAD = 1e-4    # fp32 gradients


def op_inputs(seed, Bt, L, E, N, random_A=True):
    """u, z, B, C ~ N(0,1); delta ~ 0.5 N(0,1); delta_bias = softplus^-1(dt),
    dt log-uniform [1e-3, 1e-1] (block.py:59-60); D ~ N(1, 0.1)."""
    rng = O.seeded_rng(seed)
    u = rng.standard_normal((Bt, L, E))
    delta = 0.5 * rng.standard_normal((Bt, L, E))
    z = rng.standard_normal((Bt, L, E))
    Bm = rng.standard_normal((Bt, L, N))
    Cm = rng.standard_normal((Bt, L, N))
    if random_A:
        A = -rng.uniform(0.5, float(N), size=(E, N))
    else:
        A = -np.broadcast_to(np.arange(1, N + 1, dtype=np.float64), (E, N)).copy()
    D = 1.0 + 0.1 * rng.standard_normal(E)
    dt = np.exp(rng.uniform(np.log(1e-3), np.log(1e-1), size=E))
    bias = dt + np.log(-np.expm1(-dt))
    return dict(u=u, delta=delta, A=A, B=Bm, C=Cm, D=D, z=z, delta_bias=bias)
