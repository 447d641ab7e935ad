"""LowDiff ORACLE -- test infrastructure only (see oracle/lowdiff_ref.cpp header).

numpy-facing ctypes wrapper around ``liblowdiff_ref.so``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` legs may import this package; the product package
``paper_2509_04084_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# LOWDIFF_REF_LIB: load another build of the oracle (tests/test_oracle_mutants.py loads mutants)
_LIB_PATH = os.environ.get("LOWDIFF_REF_LIB") or os.path.join(_HERE, "liblowdiff_ref.so")

OK, E_INVALID, E_DIM, E_NUMERIC, E_IO, E_CORRUPT, E_GAP = 0, 1, 2, 3, 6, 7, 8
SGD, ADAM = 0, 1
FLAG_EF, FLAG_MEAN = 1, 2


def build() -> str:
    if not os.environ.get("LOWDIFF_REF_LIB"):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        L.lowdiff_ref_k.restype = C.c_uint64
        L.lowdiff_ref_k.argtypes = [C.c_uint64, C.c_uint32]
        L.lowdiff_ref_crc32c.restype = C.c_uint32
        L.lowdiff_ref_crc32c.argtypes = [P, C.c_uint64]
        L.lowdiff_ref_compress.argtypes = [C.c_int, P, C.c_uint32, C.c_int, P, P, P]
        L.lowdiff_ref_exchange.argtypes = [C.c_int, C.c_uint64, C.c_uint64, P, C.c_int, P]
        L.lowdiff_ref_adam_consts.argtypes = [C.c_double, C.c_double, C.c_double, P]
        L.lowdiff_ref_adam_consts.restype = None
        L.lowdiff_ref_step_scalars.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double, P]
        L.lowdiff_ref_step_scalars.restype = None
        L.lowdiff_ref_adam_step.argtypes = [C.c_uint64, P, P, P, P, P, P]
        L.lowdiff_ref_sgd_step.argtypes = [C.c_uint64, P, C.c_float, P]
        L.lowdiff_ref_batch_bytes.restype = C.c_int64
        L.lowdiff_ref_batch_bytes.argtypes = [C.c_int, C.c_uint64, C.c_int]
        L.lowdiff_ref_batch_serialize.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_int, P,
                                                  C.c_uint32, C.c_uint32, C.c_uint32, P, P, P, P, C.c_uint64]
        L.lowdiff_ref_full_bytes.restype = C.c_int64
        L.lowdiff_ref_full_bytes.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
        L.lowdiff_ref_full_serialize.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint32,
                                                 C.c_uint32, P, P, P, P, P, C.c_uint64]
        L.lowdiff_ref_recover.argtypes = [C.c_char_p, C.c_uint32, C.c_int, P, C.c_uint32, C.c_int64,
                                          P, P, P, P]
        L.lowdiff_ref_union_compact.argtypes = [C.c_int, C.c_uint64, C.c_uint64, P, C.c_int, C.c_uint64,
                                                C.c_uint64, P, P, C.c_uint64, P]
        L.lowdiff_ref_union_bytes.restype = C.c_int64
        L.lowdiff_ref_union_bytes.argtypes = [C.c_int, C.c_int, P]
        L.lowdiff_ref_union_serialize.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_int, P,
                                                  C.c_uint32, C.c_uint32, C.c_uint32, P, P, P, P, P, C.c_uint64]
        L.lowdiff_ref_accumulate.argtypes = [C.c_uint32, P, P, P, P, C.c_uint64, P]
        L.lowdiff_ref_accum_serialize.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_int, P,
                                                  C.c_uint32, C.c_uint32, C.c_uint32, P, P, C.c_uint64, P, P,
                                                  C.c_uint64]
        L.lowdiff_ref_recover_union.argtypes = [C.c_char_p, C.c_uint32, C.c_int, P, C.c_uint32, C.c_int64,
                                                P, P, P, P]
        L.lowdiff_ref_wasted_time.restype = C.c_double
        L.lowdiff_ref_wasted_time.argtypes = [C.c_double] * 9
        L.lowdiff_ref_optimal_config.restype = None
        L.lowdiff_ref_optimal_config.argtypes = [C.c_double] * 4 + [C.POINTER(C.c_double)] * 2
        L.lowdiff_ref_simulate.restype = None
        L.lowdiff_ref_simulate.argtypes = [C.c_double] * 11 + [C.c_uint64, P, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class OracleError(RuntimeError):
    def __init__(self, fn, code):
        super().__init__(f"{fn} -> status {code}")
        self.code = code


def _check(fn, code):
    if code != 0:
        raise OracleError(fn, code)


def fp_env_ok() -> bool:
    return bool(lib().lowdiff_ref_fp_env_ok())


def k_of(n: int, ppm: int) -> int:
    return int(lib().lowdiff_ref_k(n, ppm))


def k_table(sizes, ppm):
    return [k_of(n, ppm) for n in sizes]


def crc32c(data: bytes) -> int:
    buf = np.frombuffer(data, dtype=np.uint8) if len(data) else np.zeros(1, np.uint8)
    return int(lib().lowdiff_ref_crc32c(_p(buf), len(data)))


def compress(sizes, ppm, grad, residual=None, ef=True):
    """Returns (send u32[2K], residual' f32[Psi] or None).  Inputs are not modified."""
    numel = _c(sizes, np.int64)
    g = _c(grad, np.float32)
    r = _c(residual, np.float32).copy() if ef else None
    K = sum(k_table(sizes, ppm))
    send = np.zeros(2 * K, np.uint32)
    _check("compress", lib().lowdiff_ref_compress(len(sizes), _p(numel), ppm, int(bool(ef)), _p(g), _p(r), _p(send)))
    return send, r


def exchange(gathered, world, K, psi, mean=True):
    ga = _c(gathered, np.uint32)
    assert ga.size == world * 2 * K
    out = np.zeros(psi, np.float32)
    _check("exchange", lib().lowdiff_ref_exchange(world, K, psi, _p(ga), int(bool(mean)), _p(out)))
    return out


def adam_consts(beta1=0.9, beta2=0.999, eps=1e-8):
    out = np.zeros(5, np.float32)
    lib().lowdiff_ref_adam_consts(beta1, beta2, eps, _p(out))
    return out


def step_scalars(t, lr, beta1=0.9, beta2=0.999):
    out = np.zeros(3, np.float32)
    lib().lowdiff_ref_step_scalars(t, lr, beta1, beta2, _p(out))
    return out


def adam_step(G, consts, scal, p, m, v):
    """In-place on p, m, v (float32 contiguous arrays)."""
    for a in (p, m, v):
        assert a.dtype == np.float32 and a.flags.c_contiguous
    Gc = _c(G, np.float32)
    _check("adam_step", lib().lowdiff_ref_adam_step(p.size, _p(Gc), _p(_c(consts, np.float32)),
                                                    _p(_c(scal, np.float32)), _p(p), _p(m), _p(v)))


def sgd_step(G, lr, p):
    assert p.dtype == np.float32 and p.flags.c_contiguous
    Gc = _c(G, np.float32)
    _check("sgd_step", lib().lowdiff_ref_sgd_step(p.size, _p(Gc), C.c_float(lr), _p(p)))


def batch_bytes(n_layers, K, n_iters):
    return int(lib().lowdiff_ref_batch_bytes(n_layers, K, n_iters))


def batch_serialize(rank, world, first_iter, sizes, ppm, optim, flags, consts, scalars, blocks) -> bytes:
    numel = _c(sizes, np.int64)
    K = sum(k_table(sizes, ppm))
    sc = _c(scalars, np.float32).reshape(-1, 3)
    bl = _c(blocks, np.uint32).reshape(-1, 2 * K)
    n = sc.shape[0]
    assert bl.shape[0] == n
    cap = batch_bytes(len(sizes), K, n)
    out = np.zeros(cap, np.uint8)
    _check("batch_serialize", lib().lowdiff_ref_batch_serialize(
        rank, world, first_iter, n, len(sizes), _p(numel), ppm, optim, flags,
        _p(_c(consts, np.float32)), _p(sc), _p(bl), _p(out), cap))
    return out.tobytes()


def full_bytes(psi, rank, world):
    return int(lib().lowdiff_ref_full_bytes(psi, rank, world))


def full_serialize(rank, world, iteration, optim, flags, consts, p, m=None, v=None) -> bytes:
    psi = int(np.asarray(p).size)
    cap = full_bytes(psi, rank, world)
    out = np.zeros(cap, np.uint8)
    pc = _c(p, np.float32)
    mc = None if m is None else _c(m, np.float32)
    vc = None if v is None else _c(v, np.float32)
    _check("full_serialize", lib().lowdiff_ref_full_serialize(
        rank, world, iteration, psi, optim, flags, _p(_c(consts, np.float32)), _p(pc), _p(mc), _p(vc),
        _p(out), cap))
    return out.tobytes()


def batch_name(rank, first):
    return f"ld_diff_r{rank:03d}_{first:012d}.ldb"


def full_name(rank, it):
    return f"ld_full_r{rank:03d}_{it:012d}.ldf"


def recover(directory, world, sizes, ppm, target=-1, with_moments=True):
    """Returns (p, m, v, recovered_iteration); m, v are None when with_moments is False."""
    numel = _c(sizes, np.int64)
    psi = int(numel.sum())
    p = np.zeros(psi, np.float32)
    m = np.zeros(psi, np.float32) if with_moments else None
    v = np.zeros(psi, np.float32) if with_moments else None
    rec = np.zeros(1, np.int64)
    _check("recover", lib().lowdiff_ref_recover(str(directory).encode(), world, len(sizes), _p(numel), ppm,
                                                target, _p(p), _p(m), _p(v), _p(rec)))
    return p, m, v, int(rec[0])


def union_compact(gathered, world, K, psi, lo=0, hi=None, mean=True):
    """Union-compacted differential C^U_t of [lo, hi): (idx u32[U], val u32[U]) -- see lowdiff_ref.cpp."""
    hi = psi if hi is None else hi
    ga = _c(gathered, np.uint32)
    assert ga.size == world * 2 * K
    cap = min(world * K, hi - lo)
    idx = np.zeros(max(cap, 1), np.uint32)
    val = np.zeros(max(cap, 1), np.uint32)
    cnt = np.zeros(1, np.uint64)
    _check("union_compact", lib().lowdiff_ref_union_compact(world, K, psi, _p(ga), int(bool(mean)), lo, hi,
                                                            _p(idx), _p(val), cap, _p(cnt)))
    n = int(cnt[0])
    return idx[:n].copy(), val[:n].copy()


def union_bytes(n_layers, counts):
    c = _c(counts, np.uint64)
    return int(lib().lowdiff_ref_union_bytes(n_layers, c.size, _p(c)))


def union_serialize(rank, world, first_iter, sizes, ppm, optim, flags, consts, scalars, unions) -> bytes:
    """unions: list of (idx, val) per iteration (this rank's shard)."""
    numel = _c(sizes, np.int64)
    sc = _c(scalars, np.float32).reshape(-1, 3)
    n = sc.shape[0]
    assert len(unions) == n
    counts = np.array([len(u[0]) for u in unions], np.uint64)
    ent = np.concatenate([np.concatenate([_c(i, np.uint32), _c(v, np.uint32)]) for i, v in unions]
                         + [np.zeros(0, np.uint32)])
    cap = union_bytes(len(sizes), counts)
    out = np.zeros(cap, np.uint8)
    _check("union_serialize", lib().lowdiff_ref_union_serialize(
        rank, world, first_iter, n, len(sizes), _p(numel), ppm, optim, flags, _p(_c(consts, np.float32)),
        _p(sc), _p(counts), _p(ent if ent.size else np.zeros(1, np.uint32)), _p(out), cap))
    return out.tobytes()


def accumulate(unions):
    """Accumulated batch mode (R-30): tensor addition of the dictionaries [(idx, val), ...] of one
    batch in iteration order -> (idx u32[A], val u32[A]) -- see lowdiff_ref.cpp."""
    counts = np.array([len(u[0]) for u in unions], np.uint64)
    ent = np.concatenate([np.concatenate([_c(i, np.uint32), _c(v, np.uint32)]) for i, v in unions]
                         + [np.zeros(1, np.uint32)])
    cap = int(counts.sum())
    idx = np.zeros(max(cap, 1), np.uint32)
    val = np.zeros(max(cap, 1), np.uint32)
    cnt = np.zeros(1, np.uint64)
    _check("accumulate", lib().lowdiff_ref_accumulate(len(unions), _p(counts if counts.size else np.zeros(1, np.uint64)),
                                                      _p(ent), _p(idx), _p(val), cap, _p(cnt)))
    n = int(cnt[0])
    return idx[:n].copy(), val[:n].copy()


def accum_serialize(rank, world, first_iter, n_iters, sizes, ppm, optim, flags, consts, last_scalars, acc) -> bytes:
    """Accumulated .ldu of one batch of n_iters iterations: acc = (idx, val) from accumulate()."""
    numel = _c(sizes, np.int64)
    idx, val = acc
    n = len(idx)
    iv = np.concatenate([_c(idx, np.uint32), _c(val, np.uint32), np.zeros(1, np.uint32)])
    cap = union_bytes(len(sizes), np.array([n], np.uint64))
    out = np.zeros(cap, np.uint8)
    _check("accum_serialize", lib().lowdiff_ref_accum_serialize(
        rank, world, first_iter, n_iters, len(sizes), _p(numel), ppm, optim, flags, _p(_c(consts, np.float32)),
        _p(_c(last_scalars, np.float32)), n, _p(iv), _p(out), cap))
    return out.tobytes()


def union_name(rank, first):
    return f"ld_union_r{rank:03d}_{first:012d}.ldu"


def recover_union(directory, world, sizes, ppm, target=-1, with_moments=True):
    """Recovery from .ldf + .ldu files: (p, m, v, recovered_iteration)."""
    numel = _c(sizes, np.int64)
    psi = int(numel.sum())
    p = np.zeros(psi, np.float32)
    m = np.zeros(psi, np.float32) if with_moments else None
    v = np.zeros(psi, np.float32) if with_moments else None
    rec = np.zeros(1, np.int64)
    _check("recover_union", lib().lowdiff_ref_recover_union(str(directory).encode(), world, len(sizes), _p(numel),
                                                            ppm, target, _p(p), _p(m), _p(v), _p(rec)))
    return p, m, v, int(rec[0])


def wasted_time(N, M, W, S, T, R_F, R_D, f, b):
    """Eq. 3, term by term (see oracle/lowdiff_ref.cpp)."""
    return float(lib().lowdiff_ref_wasted_time(N, M, W, S, T, R_F, R_D, f, b))


def optimal_config(M, W, S, R_D):
    """Eq. 5."""
    f, b = C.c_double(), C.c_double()
    lib().lowdiff_ref_optimal_config(M, W, S, R_D, C.byref(f), C.byref(b))
    return f.value, b.value


def simulate(N, M, W, S, T, R_F, R_D, f, b, sw_fraction=0.0, R_S=0.0, seed=0):
    """Failure-injection simulator: (failures, hw_failures, lost, recovery, steady, wasted)."""
    counts = np.zeros(2, np.int64)
    ledger = np.zeros(4, np.float64)
    lib().lowdiff_ref_simulate(N, M, W, S, T, R_F, R_D, f, b, sw_fraction, R_S, seed, _p(counts), _p(ledger))
    return int(counts[0]), int(counts[1]), *[float(x) for x in ledger]
