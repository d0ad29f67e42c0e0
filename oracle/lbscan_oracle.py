"""CPU restatement of the reference LB-scan path — TEST INFRASTRUCTURE ONLY.

This module is the parity *checker*.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product path (``paper_2506_15976_b200``) never imports or calls it and
fails loudly when its CUDA library is missing.

Parity pinning: every function below restates one reference function (cited as
``file:line`` relative to ``/root/reference/pkg/src/lbscan``).  The restatement
is checked against golden vectors produced by running the UNMODIFIED reference
(``oracle/gen_golden.py`` -> ``tests/golden/*.npz``) in
``tests/test_oracle_golden.py``.

Everything is float64 numpy.  Loops run over the sequence axis only; every
(b, e, n) lane is vectorised, which is exact because lanes are independent
(``engine.py:94-99``).

Layouts follow the reference (``core.py:8-14``): sequence tensors are
channel-last ``(B, L, E)``, the pre-discretised coefficients ``(B, L, E, N)``,
``c``/``B``/``C`` are ``(B, L, N)``, ``A`` is ``(E, N)``, the state ``(B, E, N)``.
"""

from __future__ import annotations

import numpy as np

RMS_EPS = 1e-6  # nn.py:13


class ShapeError(ValueError):
    """core.py:24-25"""


class NonFiniteError(ValueError):
    """core.py:28-29"""


# --------------------------------------------------------------------------
# tiling rule


def select_tile_len(L: int) -> int:
    """engine.py:54-62 — M=16 if L>256, 8 if L>128, else 4."""
    if L < 1:
        raise ShapeError(f"sequence length must be >= 1, got {L}")
    if L > 256:
        return 16
    if L > 128:
        return 8
    return 4


def tile_end(i: int, L: int, M: int) -> int:
    """oracle.py:132-138."""
    return min(L - 1, M * (i // M + 1) - 1)


def seeded_rng(seed: int) -> np.random.Generator:
    """core.py:63-65 (PCG64)."""
    return np.random.default_rng(np.random.PCG64(seed))


def random_scan_params(rng, B, L, E, N, dtype=np.float64, abar_low=0.2, abar_high=0.99):
    """core.py:131-146 — same draw order, so identical seeds give identical arrays."""
    abar = rng.uniform(abar_low, abar_high, size=(B, L, E, N)).astype(dtype)
    bx = rng.standard_normal((B, L, E, N)).astype(dtype)
    c = rng.standard_normal((B, L, N)).astype(dtype)
    dx = rng.standard_normal((B, L, E)).astype(dtype)
    return abar, bx, c, dx


def max_rel_err(got, ref, floor: float = 1e-30) -> float:
    """core.py:149-156 — inf-norm error over max |ref|."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = max(float(np.max(np.abs(ref))) if ref.size else 0.0, floor)
    if not ref.size:
        return 0.0
    return float(np.max(np.abs(got - ref))) / scale


# --------------------------------------------------------------------------
# pre-discretised scans (oracle.py)


def _f64(*arrs):
    return [np.asarray(a, dtype=np.float64) for a in arrs]


def _check_scan_shapes(abar, bx, c, dx):
    if abar.ndim != 4:
        raise ShapeError(f"abar must be (B, L, E, N), got {abar.shape}")
    B, L, E, N = abar.shape
    if bx.shape != abar.shape:
        raise ShapeError(f"bx has shape {bx.shape}, expected {abar.shape}")
    if c.shape != (B, L, N):
        raise ShapeError(f"c has shape {c.shape}, expected {(B, L, N)}")
    if dx.shape != (B, L, E):
        raise ShapeError(f"dx has shape {dx.shape}, expected {(B, L, E)}")


def forward_states(abar, bx):
    """oracle.py:39-52 state recurrence h_t = abar_t h_{t-1} + bx_t, h_{-1}=0."""
    abar, bx = _f64(abar, bx)
    B, L, E, N = abar.shape
    states = np.empty((B, L, E, N))
    h = np.zeros((B, E, N))
    for t in range(L):
        h = abar[:, t] * h + bx[:, t]
        states[:, t] = h
    return states


def forward_scan(abar, bx, c, dx):
    """oracle.py:39-52 -> (y (B,L,E), h_final (B,E,N))."""
    abar, bx, c, dx = _f64(abar, bx, c, dx)
    _check_scan_shapes(abar, bx, c, dx)
    states = forward_states(abar, bx)
    y = np.einsum("blen,bln->ble", states, c) + dx
    return y, states[:, -1].copy()


def local_backward(abar, bx, M: int):
    """oracle.py:80-112 — exclusive tile-local backward record.

    Scans i = L-1..0; the state resets to 0 where (i+1) % M == 0 and the value
    recorded at i is taken *before* bx_i is added (so it is 0 at tile ends)."""
    abar, bx = _f64(abar, bx)
    if not isinstance(M, (int, np.integer)) or M < 1:
        raise ShapeError(f"tile length M must be a positive integer, got {M!r}")
    B, L, E, N = abar.shape
    rec = np.empty((B, L, E, N))
    h = np.zeros((B, E, N))
    for i in range(L - 1, -1, -1):
        if (i + 1) % M == 0:
            h = np.zeros((B, E, N))
        else:
            h = abar[:, i] * h
        rec[:, i] = h
        h = h + bx[:, i]
    return rec


def lbm_scan(abar, bx, c, dx, M: int, return_states: bool = False):
    """oracle.py:115-129 -> (y, h_final[, h+r])."""
    abar, bx, c, dx = _f64(abar, bx, c, dx)
    _check_scan_shapes(abar, bx, c, dx)
    states = forward_states(abar, bx)
    h_sum = states + local_backward(abar, bx, M)
    y = np.einsum("blen,bln->ble", h_sum, c) + dx
    if return_states:
        return y, states[:, -1].copy(), h_sum
    return y, states[:, -1].copy()


def global_backward_scan(abar, bx, c, dx):
    """oracle.py:55-68 — right-to-left sweep."""
    flip = lambda a: np.asarray(a, np.float64)[:, ::-1]
    y, hf = forward_scan(flip(abar), flip(bx), flip(c), flip(dx))
    return y[:, ::-1].copy(), hf


def global_bidir_scan(pf, pb):
    """oracle.py:71-77 — two independent sweeps, summed."""
    yf, hf = forward_scan(*pf)
    yb, hb = global_backward_scan(*pb)
    return yf + yb, hf + hb


def lbm_scan_grad(abar, bx, c, gy, M: int, local: bool = True):
    """autodiff.py:48-159 (restated per lane, vectorised) -> (g_abar, g_bx, g_c, g_dx).

    forward part: lam_t = g_t + a_{t+1} lam_{t+1}; d bx_t += lam_t; d abar_t += lam_t h_{t-1}
    local part (ascending in each tile): v_lo = g_lo, v_i = g_i + a_{i-1} v_{i-1};
      d abar_i += v_i (r_{i+1} + bx_{i+1}) and d bx_{i+1} += a_i v_i for i < tile end
    d c_t[n] = sum_e gy_t[e] (h + r)_t[e, n]; d dx = gy   (autodiff.py:11-19)
    """
    abar, bx, c, gy = _f64(abar, bx, c, gy)
    B, L, E, N = abar.shape
    g = c[:, :, None, :] * gy[..., None]
    h = forward_states(abar, bx)
    r = local_backward(abar, bx, M) if local else np.zeros_like(h)
    ga = np.zeros_like(abar)
    gb = np.zeros_like(bx)
    lam = np.zeros((B, E, N))
    for t in range(L - 1, -1, -1):
        lam = g[:, t] + (abar[:, t + 1] * lam if t + 1 < L else 0.0)
        gb[:, t] += lam
        if t > 0:
            ga[:, t] += lam * h[:, t - 1]
    if local:
        for lo in range(0, L, M):
            hi = min(L, lo + M)
            v = None
            for i in range(lo, hi - 1):
                v = g[:, i] if i == lo else g[:, i] + abar[:, i - 1] * v
                ga[:, i] += v * (r[:, i + 1] + bx[:, i + 1])
                gb[:, i + 1] += abar[:, i] * v
    gc = np.einsum("blen,ble->bln", h + r, gy)
    return ga, gb, gc, gy.copy()


# --------------------------------------------------------------------------
# dense primitives (nn.py)


def sigmoid(x):
    """nn.py:16-18 (tanh form)."""
    return 0.5 * (1.0 + np.tanh(0.5 * x))


def softplus(x):
    """nn.py:21-22."""
    return np.logaddexp(0.0, x)


def silu(x):
    """nn.py:25-26."""
    return x * sigmoid(x)


def silu_grad(x):
    """nn.py:29-31."""
    s = sigmoid(x)
    return s * (1.0 + x * (1.0 - s))


def gelu(x):
    """nn.py:37-39 (tanh approximation)."""
    return 0.5 * x * (1.0 + np.tanh(np.sqrt(2.0 / np.pi) * (x + 0.044715 * x**3)))


def rms_norm(x, scale):
    """nn.py:55-58."""
    inv = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + RMS_EPS)
    return x * inv * scale


def causal_conv1d(x, kernel):
    """nn.py:87-99 — out[b,l,e] = sum_q kernel[e,q] x[b,l-q,e], zero left pad.

    NB: the reference tap index q counts *backwards in time*; a torch
    depthwise Conv1d weight w[e,0,j] equals kernel[e, k-1-j]."""
    x = np.asarray(x, np.float64)
    B, L, E = x.shape
    k = kernel.shape[1]
    out = np.zeros_like(x)
    for q in range(min(k, L)):
        seg = x[:, : L - q] if q else x
        out[:, q:] += kernel[:, q] * seg
    return out


def causal_conv1d_grad(x, kernel, g):
    """nn.py:102-114 -> (g_x, g_kernel)."""
    x = np.asarray(x, np.float64)
    g = np.asarray(g, np.float64)
    B, L, E = x.shape
    k = kernel.shape[1]
    g_x = np.zeros_like(x)
    g_k = np.zeros_like(kernel, dtype=np.float64)
    for q in range(min(k, L)):
        if q:
            g_x[:, : L - q] += kernel[:, q] * g[:, q:]
            g_k[:, q] = np.sum(g[:, q:] * x[:, : L - q], axis=(0, 1))
        else:
            g_x += kernel[:, 0] * g
            g_k[:, 0] = np.sum(g * x, axis=(0, 1))
    return g_x, g_k


# --------------------------------------------------------------------------
# the fused operator (north-star API) = block.py:90-98 + engine + block.py:177-178


def _flipL(a):
    return None if a is None else np.asarray(a, np.float64)[:, ::-1]


def discretize(u, delta, A, Bm, D=None, delta_bias=None, delta_softplus=True, mode="exp"):
    """block.py:87-103 with the projections already applied:
    u = x_conv, delta = x_conv @ w_delta (pre-bias), A = -exp(a_log), Bm = x_conv @ w_b.
    Returns (abar, bx, dx, dl) with dl the post-softplus step."""
    u, delta, A, Bm = _f64(u, delta, A, Bm)
    d = delta + (0.0 if delta_bias is None else np.asarray(delta_bias, np.float64))
    dl = softplus(d) if delta_softplus else d
    dA = dl[..., None] * A
    abar = np.exp(dA) if mode == "exp" else dA
    bx = dl[..., None] * Bm[:, :, None, :] * u[..., None]
    dx = (np.asarray(D, np.float64) * u) if D is not None else np.zeros_like(u)
    return abar, bx, dx, dl


def lbm_selective_scan(u, delta, A, B, C, D=None, z=None, delta_bias=None,
                       delta_softplus=True, window=None, reverse=False,
                       return_last_state=False, mode="exp", lb=True):
    """Fused LB selective scan in the reference's layout.

    u, delta, z: (Bt, L, E); A: (E, N); B, C: (Bt, L, N); D, delta_bias: (E,).
    ``reverse`` scans right-to-left with tiles aligned from the right end
    (engine.py:133,183 flip-on-load; block.py:180-181 reverse copies).
    ``lb=False`` gives the forward-only scan (engine.forward_scan_par)."""
    u = np.asarray(u, np.float64)
    L = u.shape[1]
    M = select_tile_len(L) if window is None else int(window)
    if M < 1:
        raise ShapeError(f"tile length must be >= 1, got {M}")
    if reverse:
        u, delta, B, C, z = _flipL(u), _flipL(delta), _flipL(B), _flipL(C), _flipL(z)
    abar, bx, dx, _ = discretize(u, delta, A, B, D, delta_bias, delta_softplus, mode)
    if lb:
        y, hf = lbm_scan(abar, bx, C, dx, M)
    else:
        y, hf = forward_scan(abar, bx, C, dx)
    out = y * silu(np.asarray(z, np.float64)) if z is not None else y
    if reverse:
        out = out[:, ::-1]
    out = np.ascontiguousarray(out)
    return (out, hf) if return_last_state else out


def lbm_selective_scan_bwd(dout, u, delta, A, B, C, D=None, z=None, delta_bias=None,
                           delta_softplus=True, window=None, reverse=False, mode="exp",
                           lb=True):
    """Adjoint of :func:`lbm_selective_scan` — autodiff.lbm_scan_grad
    (autodiff.py:192-195) chained through block._discretize_backward
    (block.py:106-129) and the gate (block.py:199-200).

    Returns dict du, ddelta, dA, dB, dC, dD, dz, ddelta_bias (None where the
    input was None)."""
    u = np.asarray(u, np.float64)
    L = u.shape[1]
    M = select_tile_len(L) if window is None else int(window)
    dout = np.asarray(dout, np.float64)
    if reverse:
        u, delta, B, C, z, dout = (_flipL(u), _flipL(delta), _flipL(B), _flipL(C),
                                   _flipL(z), _flipL(dout))
    A = np.asarray(A, np.float64)
    Bm = np.asarray(B, np.float64)
    abar, bx, dx, dl = discretize(u, delta, A, Bm, D, delta_bias, delta_softplus, mode)
    if z is not None:
        z = np.asarray(z, np.float64)
        y, _ = lbm_scan(abar, bx, C, dx, M) if lb else forward_scan(abar, bx, C, dx)
        gy = dout * silu(z)
        dz = dout * y * silu_grad(z)
    else:
        gy = dout
        dz = None
    ga, gb, gc, gdx = lbm_scan_grad(abar, bx, C, gy, M if lb else 1, local=lb)
    Dv = np.zeros(u.shape[-1]) if D is None else np.asarray(D, np.float64)
    du = Dv * gdx + np.einsum("blen,ble,bln->ble", gb, dl, Bm)
    t = ga * abar if mode == "exp" else ga
    ddl = np.einsum("blen,bln,ble->ble", gb, Bm, u) + np.einsum("blen,en->ble", t, A)
    d = delta + (0.0 if delta_bias is None else np.asarray(delta_bias, np.float64))
    ddelta = ddl * sigmoid(d) if delta_softplus else ddl
    out = dict(
        du=du,
        ddelta=ddelta,
        dA=np.einsum("blen,ble->en", t, dl),
        dB=np.einsum("blen,ble,ble->bln", gb, dl, u),
        dC=gc,
        dD=None if D is None else np.sum(gdx * u, axis=(0, 1)),
        dz=dz,
        ddelta_bias=None if delta_bias is None else np.sum(ddelta, axis=(0, 1)),
    )
    if reverse:
        for k in ("du", "ddelta", "dB", "dC", "dz"):
            if out[k] is not None:
                out[k] = np.ascontiguousarray(out[k][:, ::-1])
    return out


# --------------------------------------------------------------------------
# block and model (block.py / model.py) — callers of the hot path

BLOCK_FIELDS = ("norm_scale", "w_x", "w_z", "conv_kernel", "w_b", "w_c",
                "w_delta", "delta_bias", "a_log", "d_param", "w_out")


def init_block_weights(rng, D, E, N, conv_width=4):
    """block.py:52-73 — same draw order as the reference."""
    def proj(d_in, d_out):
        return rng.standard_normal((d_in, d_out)) / np.sqrt(d_in)

    dt = np.exp(rng.uniform(np.log(1e-3), np.log(1e-1), size=E))
    delta_bias = dt + np.log(-np.expm1(-dt))
    return dict(
        norm_scale=np.ones(D), w_x=proj(D, E), w_z=proj(D, E),
        conv_kernel=rng.uniform(-1, 1, size=(E, conv_width)) / np.sqrt(conv_width),
        w_b=proj(E, N), w_c=proj(E, N), w_delta=proj(E, E) * 0.1,
        delta_bias=delta_bias,
        a_log=np.broadcast_to(np.log(np.arange(1, N + 1, dtype=np.float64)), (E, N)).copy(),
        d_param=np.ones(E), w_out=proj(E, D),
    )


def block_forward(T_in, w: dict, M: int, reverse: bool = True, mode: str = "exp",
                  return_intermediates: bool = False):
    """block.py:158-190 (scan_impl="seq")."""
    T_in = np.asarray(T_in, np.float64)
    xn = rms_norm(T_in, w["norm_scale"])
    x = xn @ w["w_x"]
    z = xn @ w["w_z"]
    xc = causal_conv1d(x, w["conv_kernel"])
    xs = silu(xc)
    A = -np.exp(w["a_log"])
    out_g = lbm_selective_scan(
        xs, xs @ w["w_delta"], A, xs @ w["w_b"], xs @ w["w_c"], D=w["d_param"], z=z,
        delta_bias=w["delta_bias"], window=M, mode=mode,
    )
    out = out_g @ w["w_out"] + T_in
    if reverse:
        out = out[:, ::-1].copy()
    if return_intermediates:
        return out, dict(xn=xn, x=x, z=z, xc=xc, xs=xs, yg=out_g)
    return out


CLASS_TOKEN_COUNT = {"none": 0, "head": 1, "middle": 1, "double": 2}


def patchify(images, patch):
    """model.py:155-161."""
    B, H, W, C = images.shape
    gh, gw = H // patch, W // patch
    x = images.reshape(B, gh, patch, gw, patch, C).transpose(0, 1, 3, 2, 4, 5)
    return x.reshape(B, gh * gw, patch * patch * C)


def insert_class_token(tokens, cls, mode):
    """model.py:164-177."""
    B, L, D = tokens.shape
    tile = lambda i: np.broadcast_to(cls[i], (B, 1, D))
    if mode == "none":
        return tokens
    if mode == "head":
        return np.concatenate([tile(0), tokens], axis=1)
    if mode == "middle":
        mid = L // 2
        return np.concatenate([tokens[:, :mid], tile(0), tokens[:, mid:]], axis=1)
    return np.concatenate([tile(0), tokens, tile(1)], axis=1)


def class_token_positions(mode, num_patches, seq_len):
    """model.py:180-187."""
    if mode == "none":
        return []
    if mode == "head":
        return [0]
    if mode == "middle":
        return [num_patches // 2]
    return [0, seq_len - 1]


def reversal_invariant_mean(tokens):
    """nn.py:117-131."""
    L = tokens.shape[1]
    half = L // 2
    front = tokens[:, :half]
    back = tokens[:, L - 1: L - 1 - half: -1] if half else tokens[:, :0]
    total = np.sum(front + back, axis=1)
    if L % 2:
        total = total + tokens[:, half]
    return total / L


def softmax(x, axis=-1):
    s = x - np.max(x, axis=axis, keepdims=True)
    e = np.exp(s)
    return e / np.sum(e, axis=axis, keepdims=True)


def model_forward(images, cfg: dict, params: dict):
    """model.py:287-325 (scan_impl="seq").  ``cfg`` keys follow ModelConfig
    (model.py:25-43): image_size, patch_size, in_channels, embed_dim,
    inner_dim, state_dim, depth, tile_len, head, map_heads, class_token,
    reverse_between_blocks, unreverse_output, discretize_mode."""
    images = np.asarray(images, np.float64)
    p = cfg["patch_size"]
    grid = cfg["image_size"] // p
    num_patches = grid * grid
    ct = cfg.get("class_token", "none")
    seq_len = num_patches + CLASS_TOKEN_COUNT[ct]
    M = cfg.get("tile_len") or select_tile_len(seq_len)
    rev = cfg.get("reverse_between_blocks", True)
    tokens = patchify(images, p) @ params["patch_w"] + params["patch_b"]
    if CLASS_TOKEN_COUNT[ct]:
        tokens = insert_class_token(tokens, params["cls"], ct)
    tokens = tokens + params["pos"]
    for i in range(cfg["depth"]):
        w = {f: params[f"blocks.{i}.{f}"] for f in BLOCK_FIELDS}
        tokens = block_forward(tokens, w, M, reverse=rev, mode=cfg.get("discretize_mode", "exp"))
    final_flip = False
    if rev and cfg["depth"] % 2 == 1 and cfg.get("unreverse_output", True):
        tokens = tokens[:, ::-1].copy()
        final_flip = True
    in_order = (not rev) or cfg["depth"] % 2 == 0 or final_flip
    if ct != "none":
        pos = class_token_positions(ct, num_patches, seq_len)
        L = tokens.shape[1]
        idx = pos if in_order else [L - 1 - q for q in pos]
        pooled = tokens[:, idx].mean(axis=1)
    elif cfg.get("head", "gap") == "gap":
        pooled = reversal_invariant_mean(tokens)
    else:
        B, L, Dm = tokens.shape
        nh = cfg["map_heads"]
        dh = Dm // nh
        K = (tokens @ params["head.wk"]).reshape(B, L, nh, dh)
        V = (tokens @ params["head.wv"]).reshape(B, L, nh, dh)
        q = params["head.q"].reshape(nh, dh)
        att = softmax(np.einsum("blhd,hd->blh", K, q) / np.sqrt(dh), axis=1)
        pooled = np.einsum("blh,blhd->bhd", att, V).reshape(B, Dm)
    h1 = gelu(pooled @ params["head.mlp_w1"] + params["head.mlp_b1"])
    return h1 @ params["head.mlp_w2"] + params["head.mlp_b2"]
