"""fp64 attention oracle (TEST INFRASTRUCTURE ONLY) -- ctypes front end of attention_oracle.c.

Definition followed (Alg. 1 line 3 ``attention(Q[:,j],K[:,j],V[:,j])``;
scale 1/sqrt(D) from BASELINE.json north_star, reading R1):

    O[b,s,k,:] = sum_t softmax_t( (sum_d Q[b,s,k,d] K[b,t,k,d]) / sqrt(D) ) V[b,t,k,:]

Inputs are float64 arrays (bf16 values converted exactly by the caller).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "attention_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def library_path() -> str:
    return _LIB


def build_library(force: bool = False) -> str:
    """gcc the plain C oracle (no -ffast-math: IEEE fp64, fixed order)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-std=c11", "-fPIC", "-shared",
               "-pthread", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build_library()
        lib = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_attention_rows.argtypes = [dp, ctypes.c_long, ctypes.c_long, dp, dp, ctypes.c_long,
                                              ctypes.c_long, dp, ctypes.c_long, ctypes.c_int]
        lib.oracle_attention_rows.restype = ctypes.c_int
        lib.oracle_softmax_weights.argtypes = [dp, dp, ctypes.c_long, ctypes.c_long, dp]
        lib.oracle_softmax_weights.restype = ctypes.c_int
        u8p = ctypes.POINTER(ctypes.c_ubyte)
        lib.oracle_attention_rows_masked.argtypes = [dp, ctypes.c_long, ctypes.c_long, dp, dp, ctypes.c_long,
                                                     ctypes.c_long, u8p, dp, ctypes.c_long, ctypes.c_int]
        lib.oracle_attention_rows_masked.restype = ctypes.c_int
        lib.oracle_attention_rows_lse.argtypes = [dp, ctypes.c_long, ctypes.c_long, dp, dp, ctypes.c_long,
                                                  ctypes.c_long, u8p, dp, ctypes.c_long, dp, ctypes.c_int]
        lib.oracle_attention_rows_lse.restype = ctypes.c_int
        _lib = lib
    return _lib


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64c(a) -> np.ndarray:
    a = np.asarray(a)
    if a.dtype != np.float64:
        raise TypeError("oracle takes float64 arrays (convert bf16 exactly first)")
    return np.ascontiguousarray(a)


def default_threads() -> int:
    return os.cpu_count() or 1


def attention_rows(q: np.ndarray, K: np.ndarray, V: np.ndarray, nthreads: Optional[int] = None,
                   key_valid: Optional[np.ndarray] = None) -> np.ndarray:
    """q [R,D], K [S,D], V [S,D] (float64) -> [R,D] float64.

    key_valid: optional [S] bool key-padding mask (Alg. 1's attention_mask; DESIGN.md
    R20): masked keys take no part in the softmax; a row with no valid key is 0."""
    q, K, V = _f64c(q), _f64c(K), _f64c(V)
    if q.ndim == 1:
        return attention_rows(q[None], K, V, nthreads, key_valid)[0]
    R, D = q.shape
    S = K.shape[0]
    assert K.shape == (S, D) and V.shape == (S, D)
    out = np.empty((R, D), dtype=np.float64)
    nt = int(nthreads or default_threads())
    if key_valid is None:
        rc = _load().oracle_attention_rows(_dptr(q), R, D, _dptr(K), _dptr(V), S, D, _dptr(out), D, nt)
    else:
        kv = np.ascontiguousarray(np.asarray(key_valid, dtype=bool).astype(np.uint8))
        assert kv.shape == (S,)
        rc = _load().oracle_attention_rows_masked(_dptr(q), R, D, _dptr(K), _dptr(V), S, D,
                                                  kv.ctypes.data_as(ctypes.POINTER(ctypes.c_ubyte)), _dptr(out),
                                                  D, nt)
    if rc != 0:
        raise RuntimeError(f"oracle_attention_rows failed ({rc})")
    return out


def attention_rows_lse(q: np.ndarray, K: np.ndarray, V: np.ndarray, nthreads: Optional[int] = None,
                       key_valid: Optional[np.ndarray] = None):
    """(O [R,D], lse [R]): attention_rows and lse[r] = ln sum_t exp(q_r . k_t / sqrt(D)) over the valid keys
    (-inf when none) -- what partial softmaxes over disjoint key blocks combine with (R21)."""
    q, K, V = _f64c(q), _f64c(K), _f64c(V)
    R, D = q.shape
    S = K.shape[0]
    out = np.empty((R, D), dtype=np.float64)
    lse = np.empty(R, dtype=np.float64)
    kvp = None
    if key_valid is not None:
        kv = np.ascontiguousarray(np.asarray(key_valid, dtype=bool).astype(np.uint8))
        kvp = kv.ctypes.data_as(ctypes.POINTER(ctypes.c_ubyte))
    rc = _load().oracle_attention_rows_lse(_dptr(q), R, D, _dptr(K), _dptr(V), S, D, kvp, _dptr(out), D, _dptr(lse),
                                           int(nthreads or default_threads()))
    if rc != 0:
        raise RuntimeError("oracle_attention_rows_lse failed")
    return out, lse


def softmax_weights(q: np.ndarray, K: np.ndarray) -> np.ndarray:
    """Softmax weights of one query row against K: [S] float64."""
    q, K = _f64c(q), _f64c(K)
    w = np.empty(K.shape[0], dtype=np.float64)
    rc = _load().oracle_softmax_weights(_dptr(q), _dptr(K), K.shape[0], K.shape[1], _dptr(w))
    if rc != 0:
        raise RuntimeError("oracle_softmax_weights failed")
    return w


def mha_unsharded(Q: np.ndarray, K: np.ndarray, V: np.ndarray, nthreads: Optional[int] = None,
                  key_valid: Optional[np.ndarray] = None) -> np.ndarray:
    """Full multi-head attention on unsharded [B,S,H,D] float64 tensors (per head, per batch).

    key_valid: optional [B,S] bool key-padding mask (the same for every head of a batch entry)."""
    B, S, H, D = Q.shape
    out = np.empty((B, S, H, D), dtype=np.float64)
    for b in range(B):
        kv = None if key_valid is None else np.asarray(key_valid)[b]
        for k in range(H):
            out[b, :, k, :] = attention_rows(np.ascontiguousarray(Q[b, :, k, :]),
                                             np.ascontiguousarray(K[b, :, k, :]),
                                             np.ascontiguousarray(V[b, :, k, :]), nthreads, kv)
    return out


def key_valid_from_lengths(kv_len, S: int) -> np.ndarray:
    """[B,S] bool mask of a key-padding length vector: key t of batch b is valid iff t < kv_len[b]."""
    kv_len = np.asarray(kv_len, dtype=np.int64)
    return np.arange(S)[None, :] < kv_len[:, None]
