"""CPU port of the reference's scan path — BASELINE / TEST INFRASTRUCTURE ONLY.

Used by bench.py's ``cpu_baseline`` leg and ``--impl reference`` arm (the
Python reference itself cannot travel to the GPU box), and by tests.  It
restates the reference's CPU pipeline:

* numpy discretisation, materialising the two (B, L, E, N) tensors exactly as
  block._discretize_cached does (block.py:87-103);
* the tiled engine (engine._scan_kernel, engine.py:88-218) as C + OpenMP
  (oracle/lbscan_ref.c), fp32 data with fp64 tile carries, all host cores;
* the gate y * silu(z) (block.py:177-178), and for the model the reference's
  numpy block / model forward (block.py:158-190, model.py:287-325).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "lbscan_ref.c")
LIB = os.path.join(HERE, "liblbscan_ref.so")

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        # no FMA contraction: the reference's numba kernel does not contract either
        cmd = ["gcc", "-O3", "-march=x86-64-v3", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
               SRC, "-o", LIB]
        subprocess.run(cmd, check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        fp = ctypes.POINTER(ctypes.c_float)
        i64 = ctypes.c_int64
        L.lbs_ref_scan_f32.argtypes = [fp, fp, fp, fp, i64, i64, i64, i64, i64, ctypes.c_int, ctypes.c_int,
                                       fp, fp, ctypes.c_int]
        L.lbs_ref_scan_f32.restype = None
        L.lbs_ref_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _fp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def scan_par(abar, bx, c, dx, M, do_backward=True, reverse=False, threads=0):
    """engine.lbm_scan_par / forward_scan_par equivalent (fp32) -> (y, h_final)."""
    abar = np.ascontiguousarray(abar, np.float32)
    B, L, E, N = abar.shape
    bx = np.ascontiguousarray(bx, np.float32)
    c = np.ascontiguousarray(c, np.float32)
    dx = np.ascontiguousarray(dx, np.float32)
    y = np.empty((B, L, E), np.float32)
    hf = np.empty((B, E, N), np.float32)
    lib().lbs_ref_scan_f32(_fp(abar), _fp(bx), _fp(c), _fp(dx), B, L, E, N, int(M), int(do_backward),
                           int(reverse), _fp(y), _fp(hf), int(threads))
    return y, hf


def num_threads() -> int:
    return int(lib().lbs_ref_num_threads())


def _softplus(x):
    return np.logaddexp(np.float32(0), x)


def _silu(x):
    return x * (np.float32(0.5) * (np.float32(1) + np.tanh(np.float32(0.5) * x)))


def fused_op(u, delta, A, B, C, D, z, delta_bias, M, reverse=False, threads=0):
    """The reference CPU composition for the fused operator (fp32):
    block.py:90-98 discretisation, engine scan, block.py:177-178 gate."""
    dl = _softplus(delta + delta_bias)
    abar = np.exp(dl[..., None] * A)
    bx = dl[..., None] * B[:, :, None, :] * u[..., None]
    y, _ = scan_par(abar, bx, C, D * u, M, True, reverse, threads)
    return y * _silu(z)


def block_forward(T, w, M, reverse_scan, threads=0):
    """block.py:158-190 in fp32 numpy + the C engine.  As on the GPU path the
    sequence stays in input order and odd blocks scan right-to-left
    (equivalent to the reference's per-block reversal)."""
    inv = 1.0 / np.sqrt(np.mean(T * T, axis=-1, keepdims=True) + np.float32(1e-6))
    xn = T * inv * w["norm_scale"]
    x = xn @ w["w_x"]
    z = xn @ w["w_z"]
    L = x.shape[1]
    k = w["conv_kernel"].shape[1]
    xr = x[:, ::-1] if reverse_scan else x
    xc = np.zeros_like(xr)
    for q in range(min(k, L)):
        xc[:, q:] += w["conv_kernel"][:, q] * (xr[:, : L - q] if q else xr)
    if reverse_scan:
        xc = xc[:, ::-1]
    xs = _silu(xc)
    A = -np.exp(w["a_log"])
    yg = fused_op(xs, xs @ w["w_delta"], A, xs @ w["w_b"], xs @ w["w_c"], w["d_param"], z,
                  w["delta_bias"], M, reverse_scan, threads)
    return yg @ w["w_out"] + T


def model_forward(images, cfg: dict, params: dict, threads=0):
    """model.py:287-325 (gap head / class-token readout), fp32."""
    p = cfg["patch_size"]
    B, H, W, C = images.shape
    g = H // p
    x = images.reshape(B, g, p, g, p, C).transpose(0, 1, 3, 2, 4, 5).reshape(B, g * g, p * p * C)
    tok = x @ params["patch_w"] + params["patch_b"]
    ct = cfg.get("class_token", "none")
    if ct == "middle":
        mid = tok.shape[1] // 2
        tok = np.concatenate([tok[:, :mid], np.broadcast_to(params["cls"][0], (B, 1, tok.shape[2])),
                              tok[:, mid:]], axis=1)
    elif ct == "head":
        tok = np.concatenate([np.broadcast_to(params["cls"][0], (B, 1, tok.shape[2])), tok], axis=1)
    tok = (tok + params["pos"]).astype(np.float32)
    L = tok.shape[1]
    M = cfg.get("tile_len") or (16 if L > 256 else 8 if L > 128 else 4)
    fields = ("norm_scale", "w_x", "w_z", "conv_kernel", "w_b", "w_c", "w_delta", "delta_bias", "a_log",
              "d_param", "w_out")
    for i in range(cfg["depth"]):
        w = {f: params[f"blocks.{i}.{f}"] for f in fields}
        tok = block_forward(tok, w, M, reverse_scan=bool(i % 2), threads=threads)
    if ct != "none":
        pooled = tok[:, [g * g // 2] if ct == "middle" else [0]].mean(axis=1)
    else:
        pooled = tok.mean(axis=1)
    h1 = pooled @ params["head.mlp_w1"] + params["head.mlp_b1"]
    h1 = 0.5 * h1 * (1 + np.tanh(np.sqrt(2 / np.pi) * (h1 + 0.044715 * h1 ** 3)))
    return h1 @ params["head.mlp_w2"] + params["head.mlp_b2"]
