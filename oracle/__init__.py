"""CPU oracle for the PP-GNN mini-batch loading hot path (arXiv 2504.13266).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package.  The product package ``paper_2504_13266_b200`` never imports it
and shares no code with it; the arithmetic lives in ``pp_oracle.c`` (plain C,
single-threaded unless a caller passes ``nthreads``), this module is ctypes
marshalling plus the plain compositions of the C steps.

Every function cites the passage it follows (PAPER.md line numbers are lines
of the paper's LaTeX source; SURVEY.md §8(c) rows O1..O11 name the steps).
Pins: see the header of ``pp_oracle.c`` and ``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

F32, BF16, F16 = 0, 1, 2
_DT = {F32: np.uint32, BF16: np.uint16, F16: np.uint16}


def build(force: bool = False) -> str:
    """Compile pp_oracle.c into liboracle.so (gcc, -O2, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i64, i32, u64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
            sig = {
                "ppo_philox4x32_10": (None, [P, P, P]),
                "ppo_unit_key": (u64, [u64, u64]),
                "ppo_unit_keys": (None, [u64, i64, P]),
                "ppo_philox_batch": (None, [P, P, i64, P]),
                "ppo_unit_key_batch": (None, [u64, P, i64, P]),
                "ppo_unit_permutation": (ctypes.c_int, [u64, i64, P]),
                "ppo_epoch_order": (ctypes.c_int, [u64, i64, i64, P]),
                "ppo_apply_node_set": (None, [P, i64, P]),
                "ppo_num_steps": (i64, [i64, i64, i32, i32]),
                "ppo_batch_range": (None, [i64, i64, i32, i64, i32, P, P]),
                "ppo_f32_to_bf16": (ctypes.c_uint16, [ctypes.c_uint32]),
                "ppo_f32_to_f16": (ctypes.c_uint16, [ctypes.c_uint32]),
                "ppo_cast_bf16_array": (None, [P, i64, P]),
                "ppo_cast_f16_array": (None, [P, i64, P]),
                "ppo_gather_cast": (ctypes.c_int, [P, i32, i64, i64, i32, i32, P, i64, i32, P, i32]),
                "ppo_gather_labels": (None, [P, P, i64, P]),
                "ppo_build_csr": (ctypes.c_int, [i64, P, P, i64, P, P, P]),
                "ppo_operator_values": (None, [i64, P, P, P]),
                "ppo_spmm": (None, [i64, i32, P, P, P, P, P]),
                "ppo_propagate": (None, [i64, i32, P, P, P, P, i32, P]),
                "ppo_gen_f32_bits": (ctypes.c_uint32, [u64, i64, i64, i64]),
                "ppo_gen_f16_bits": (ctypes.c_uint16, [u64, i64, i64, i64]),
                "ppo_gen_rows": (ctypes.c_int, [u64, i32, i32, i32, P, i64, P, i32]),
                "ppo_gen_graph": (ctypes.c_int, [u64, i64, i64, P, P]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return ctypes.c_void_p(a.ctypes.data)


# --------------------------------------------------------------------------- O4-O9: the shuffle
def philox(ctr, key) -> np.ndarray:
    """O4: Philox4x32-10 of one (ctr[4], key[2]) -> 4 x u32."""
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().ppo_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def philox_batch(ctr: np.ndarray, key: np.ndarray) -> np.ndarray:
    """O4 over many inputs: ctr [n, 4] u32, key [n, 2] u32 -> [n, 4] u32."""
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros((c.shape[0], 4), dtype=np.uint32)
    lib().ppo_philox_batch(_p(c), _p(k), c.shape[0], _p(out))
    return out


def unit_key_at(seed: int, units) -> np.ndarray:
    """O5: sort keys of arbitrary (64-bit) unit ids."""
    u = np.ascontiguousarray(units, dtype=np.uint64)
    out = np.zeros(u.shape[0], dtype=np.uint64)
    lib().ppo_unit_key_batch(seed, _p(u), u.shape[0], _p(out))
    return out


def unit_keys(seed: int, U: int) -> np.ndarray:
    """O5: 64-bit sort keys of units 0..U-1 for epoch seed ``seed``."""
    out = np.zeros(U, dtype=np.uint64)
    lib().ppo_unit_keys(seed, U, _p(out))
    return out


def unit_permutation(seed: int, U: int) -> np.ndarray:
    """O6: units sorted by (key64, unit id)."""
    out = np.zeros(U, dtype=np.int64)
    rc = lib().ppo_unit_permutation(seed, U, _p(out))
    assert rc == 0
    return out


def epoch_order(seed: int, N: int, chunk: int, node_set: np.ndarray | None = None) -> np.ndarray:
    """O7 (+O8): the epoch's visiting order of the N positions (chunk=1: SGD-RR,
    PAPER.md:70; chunk>1: chunk reshuffling).  With a node set the
    positions index into it."""
    if chunk < 1 or (N > 0 and chunk > N):
        raise ValueError("chunk must be in [1, N]")
    out = np.zeros(N, dtype=np.int64)
    rc = lib().ppo_epoch_order(seed, N, chunk, _p(out))
    assert rc == 0
    if node_set is not None:
        S = np.ascontiguousarray(node_set, dtype=np.int64)
        assert S.shape[0] == N
        lib().ppo_apply_node_set(_p(S), N, _p(out))
    return out


def num_steps(N: int, B: int, W: int = 1, drop_last: bool = False) -> int:
    """O9: steps per epoch."""
    return int(lib().ppo_num_steps(N, B, W, int(drop_last)))


def batch_range(N: int, B: int, W: int, t: int, r: int) -> tuple[int, int]:
    """O9: positions [start, end) of rank r's batch at step t."""
    s = ctypes.c_int64()
    e = ctypes.c_int64()
    lib().ppo_batch_range(N, B, W, t, r, ctypes.byref(s), ctypes.byref(e))
    return s.value, e.value


# --------------------------------------------------------------------------- O10: casts and gather
def cast_bf16(bits: np.ndarray) -> np.ndarray:
    """O10: fp32 bit patterns -> bf16 bit patterns (RNE, NaN -> 0x7FFF)."""
    b = np.ascontiguousarray(bits, dtype=np.uint32)
    out = np.zeros(b.shape, dtype=np.uint16)
    lib().ppo_cast_bf16_array(_p(b), b.size, _p(out))
    return out


def cast_f16(bits: np.ndarray) -> np.ndarray:
    """O10: fp32 bit patterns -> binary16 bit patterns (RNE, NaN -> 0x7FFF)."""
    b = np.ascontiguousarray(bits, dtype=np.uint32)
    out = np.zeros(b.shape, dtype=np.uint16)
    lib().ppo_cast_f16_array(_p(b), b.size, _p(out))
    return out


def gather_cast(X: np.ndarray, in_dtype: int, hop_stride: int, row_stride: int, H: int, F: int,
                rows: np.ndarray, out_dtype: int, nthreads: int = 1) -> np.ndarray:
    """O10: out[j, k, f] = cast(X_k[rows[j], f]), elem(k, v, f) = X.flat[k*hop_stride + v*row_stride + f].

    ``X`` is passed as raw bit patterns (uint32 for fp32, uint16 for 16-bit)."""
    Xc = np.ascontiguousarray(X)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros((r.shape[0], H, F), dtype=_DT[out_dtype])
    rc = lib().ppo_gather_cast(_p(Xc), in_dtype, hop_stride, row_stride, H, F, _p(r), r.shape[0],
                               out_dtype, _p(out), nthreads)
    if rc != 0:
        raise ValueError("unsupported dtype pair")
    return out


def gather_labels(labels: np.ndarray, rows: np.ndarray) -> np.ndarray:
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros(r.shape[0], dtype=np.int32)
    lib().ppo_gather_labels(_p(lab), _p(r), r.shape[0], _p(out))
    return out


def batch(X, in_dtype, hop_stride, row_stride, H, F, order, B, W, t, r, out_dtype, labels=None):
    """O9 + O10 composed: rank r's batch at step t -> (feat [rows,H,F], labels, node ids)."""
    s, e = batch_range(order.shape[0], B, W, t, r)
    rows = order[s:e]
    feat = gather_cast(X, in_dtype, hop_stride, row_stride, H, F, rows, out_dtype)
    lab = gather_labels(labels, rows) if labels is not None else None
    return feat, lab, rows.copy()


# --------------------------------------------------------------------------- A0: propagation (Eq. 2)
def build_csr(n: int, src, dst):
    """O1: CSR of A~ = I + A (undirected, deduplicated, one diagonal entry per row)."""
    s = np.ascontiguousarray(src, dtype=np.int64)
    d = np.ascontiguousarray(dst, dtype=np.int64)
    nnz = ctypes.c_int64()
    rp = np.zeros(n + 1, dtype=np.int64)
    rc = lib().ppo_build_csr(n, _p(s), _p(d), s.shape[0], _p(rp), None, ctypes.byref(nnz))
    if rc != 0:
        raise ValueError("bad edge list")
    ci = np.zeros(max(nnz.value, 1), dtype=np.int64)
    rc = lib().ppo_build_csr(n, _p(s), _p(d), s.shape[0], _p(rp), _p(ci), ctypes.byref(nnz))
    assert rc == 0
    return rp, ci[: nnz.value].copy()


def operator_values(n: int, row_ptr: np.ndarray, col_idx: np.ndarray) -> np.ndarray:
    """O2: B = D~^-1/2 A~ D~^-1/2 values."""
    val = np.zeros(max(col_idx.shape[0], 1), dtype=np.float64)
    lib().ppo_operator_values(n, _p(row_ptr), _p(col_idx), _p(val))
    return val[: col_idx.shape[0]].copy()


def spmm(n, row_ptr, col_idx, val, X: np.ndarray) -> np.ndarray:
    """O3: one fp64-accumulate / fp32-store SpMM."""
    Xc = np.ascontiguousarray(X, dtype=np.float32)
    F = Xc.shape[1]
    Y = np.zeros_like(Xc)
    lib().ppo_spmm(n, F, _p(row_ptr), _p(col_idx), _p(val), _p(Xc), _p(Y))
    return Y


def propagate(n: int, row_ptr, col_idx, val, X: np.ndarray, K: int) -> np.ndarray:
    """Eq. (2): hop-major [K+1, n, F] fp32 with hops[0] == X."""
    Xc = np.ascontiguousarray(X, dtype=np.float32)
    F = Xc.shape[1]
    hops = np.zeros((K + 1, n, F), dtype=np.float32)
    lib().ppo_propagate(n, F, _p(row_ptr), _p(col_idx), _p(val), _p(Xc), K, _p(hops))
    return hops


def propagate_graph(n: int, src, dst, X: np.ndarray, K: int) -> np.ndarray:
    rp, ci = build_csr(n, src, dst)
    return propagate(n, rp, ci, operator_values(n, rp, ci), X, K)


# --------------------------------------------------------------------------- O11: synthetic inputs
def gen_rows(seed: int, dtype: int, H: int, F: int, rows, nthreads: int = 1) -> np.ndarray:
    """O11: generator G (fp32) or G16 (fp16) for the given rows, node-major [rows, H, F] bits."""
    r = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros((r.shape[0], H, F), dtype=_DT[dtype])
    rc = lib().ppo_gen_rows(seed, dtype, H, F, _p(r), r.shape[0], _p(out), nthreads)
    if rc != 0:
        raise ValueError("generator supports F32 and F16 only")
    return out


def gen_graph(seed: int, n: int, m: int):
    """Config-1 Erdos-Renyi edge list."""
    src = np.zeros(m, dtype=np.int64)
    dst = np.zeros(m, dtype=np.int64)
    rc = lib().ppo_gen_graph(seed, n, m, _p(src), _p(dst))
    if rc != 0:
        raise ValueError("bad graph parameters")
    return src, dst


def tiny_hops(data_seed: int = 2504, n: int = 2708, m: int = 5429, F: int = 128, K: int = 3) -> np.ndarray:
    """Config 1: X_0 = G(data_seed) over n nodes, K hops of B by oracle SpMM -> [K+1, n, F] fp32."""
    src, dst = gen_graph(data_seed, n, m)
    X0 = gen_rows(data_seed, F32, 1, F, np.arange(n)).reshape(n, F).view(np.float32)
    return propagate_graph(n, src, dst, X0, K)


# --------------------------------------------------------------------------- §8(f)-1 consumer: per-hop linear
def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    """bf16 bit patterns -> exact float64 values (a bf16 is the top half of an fp32)."""
    return (np.asarray(bits, dtype=np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def f16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    """binary16 bit patterns -> exact float64 values."""
    return np.asarray(bits, dtype=np.uint16).view(np.float16).astype(np.float64)


def hop_linear(batch_bits: np.ndarray, W_bits: np.ndarray, dtype: int = BF16):
    """SIGN's per-hop linear layer (one weight matrix per hop) on a batch:
    Z[j, k, :] = X[j, k, :] @ W[k] in float64 from the exact 16-bit values (numpy matmul as the
    library step).  batch_bits: bf16 (dtype BF16) or binary16 (dtype F16) bits [rows, H, F] (the
    oracle batch, O10); W_bits: the same type's bits [H, F, D].  Returns (Z, S) with
    S[j, k, :] = |X[j, k, :]| @ |W[k]| (the scale of the rounding-error bound of any summation
    order)."""
    to64 = bf16_bits_to_f64 if dtype == BF16 else f16_bits_to_f64
    X = to64(batch_bits)
    Wf = to64(W_bits)
    Z = np.einsum("jkf,kfd->jkd", X, Wf)
    S = np.einsum("jkf,kfd->jkd", np.abs(X), np.abs(Wf))
    return Z, S
