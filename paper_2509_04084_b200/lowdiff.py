"""Thin Python binding of liblowdiff (include/lowdiff.h) -- argument marshalling only.

Every step of the LowDiff hot path runs in the CUDA library; this module only turns
torch tensors into device pointers, streams into cudaStream_t handles, and status codes into
exceptions.  There is no fallback: if ``_lib/liblowdiff.so`` is missing the import fails.
Function names follow the C ABI (``lowdiff_<name>`` -> ``Context.<name>``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LOWDIFF_LIB") or os.path.join(_HERE, "_lib", "liblowdiff.so")   # env: tuning builds

OK, E_INVALID, E_DIM, E_NUMERIC, E_CUDA, E_NCCL, E_IO, E_CORRUPT, E_GAP, E_STATE = range(10)
SGD, ADAM = 0, 1
BATCH_RECORD, BATCH_ACCUMULATED = 0, 1   # lowdiff_set_batch_mode
STATUS_NAMES = ["OK", "E_INVALID", "E_DIM", "E_NUMERIC", "E_CUDA", "E_NCCL", "E_IO", "E_CORRUPT",
                "E_GAP", "E_STATE"]


class LowDiffError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str = ""):
        name = STATUS_NAMES[code] if 0 <= code < len(STATUS_NAMES) else str(code)
        super().__init__(f"lowdiff_{fn} -> {name}" + (f": {msg}" if msg else ""))
        self.code = code


class StepScalars(C.Structure):
    _fields_ = [("lr", C.c_float), ("bc1_inv", C.c_float), ("bc2_inv", C.c_float)]


class AdamConsts(C.Structure):
    _fields_ = [("beta1", C.c_float), ("one_minus_beta1", C.c_float), ("beta2", C.c_float),
                ("one_minus_beta2", C.c_float), ("eps", C.c_float)]


class Config(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("numel", C.POINTER(C.c_int64)), ("density_ppm", C.c_uint32),
                ("error_feedback", C.c_int32), ("mean", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("nccl_unique_id", C.c_void_p), ("device", C.c_int32), ("ckpt_dir", C.c_char_p),
                ("batch_size", C.c_int32), ("ring_slots", C.c_int32), ("write_files", C.c_int32),
                ("fsync", C.c_int32), ("optim", C.c_int32), ("adam", AdamConsts)]


class SysParams(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("N", "M", "W", "S", "T", "R_F", "R_D")]


class SimReport(C.Structure):
    _fields_ = [("failures", C.c_int64), ("hw_failures", C.c_int64), ("lost_work", C.c_double),
                ("recovery", C.c_double), ("steady", C.c_double), ("wasted", C.c_double),
                ("effective_ratio", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("files_written", C.c_int64), ("bytes_written", C.c_int64), ("ring_stall_ns", C.c_int64),
                ("writer_busy_ns", C.c_int64), ("spec_hits", C.c_int64), ("spec_misses", C.c_int64),
                ("spec_candidates", C.c_int64), ("replica_busy_ns", C.c_int64), ("replica_stall_ns", C.c_int64),
                ("union_files_written", C.c_int64), ("union_bytes_written", C.c_int64), ("union_entries", C.c_int64),
                ("direct_segments", C.c_int64), ("compress_scratch_bytes", C.c_int64), ("device_bytes", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        P, S = C.c_void_p, C.c_int
        sig = {
            "create": ([C.POINTER(Config), C.POINTER(C.c_void_p)], S),
            "destroy": ([P], S),
            "query": ([P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], S),
            "layer_k": ([P, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], S),
            "compress": ([P, P, P, P, P], S),
            "residual_materialize": ([P, P, P], S),
            "exchange": ([P, P, P, P, P], S),
            "merge": ([P, C.c_int32, P, P, P], S),
            "exchange_update": ([P, P, P, C.POINTER(StepScalars), P, P, P, P], S),
            "peer_alloc": ([P, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), P], S),
            "ipc_open": ([P, P, C.POINTER(C.c_void_p)], S),
            "peer_set": ([P, C.POINTER(C.c_void_p)], S),
            "exchange_peer": ([P, C.c_int32, P, P], S),
            "exchange_peer_update": ([P, C.c_int32, C.POINTER(StepScalars), P, P, P, P], S),
            "batch_persist": ([P, C.c_int64, C.POINTER(StepScalars), P, P], S),
            "full_ckpt": ([P, C.c_int64, P, P, P, P], S),
            "wait_persist": ([P, P], S),
            "recover": ([P, C.c_int64, P, P, P, C.POINTER(C.c_int64), P], S),
            "replay": ([P, C.c_int32, C.c_int32, C.c_int64, P, P, P, P, P, P], S),
            "replay_range": ([P, C.c_int32, C.c_int32, C.c_int64, P, P, C.c_int64, C.c_int64, P, P, P, P], S),
            "recover_sharded": ([P, C.c_int64, P, P, P, C.c_int32, C.POINTER(C.c_int64), P], S),
            "snapshot_layer": ([P, C.c_int64, C.c_int32, C.c_int32, P, P], S),
            "snapshot_wait": ([P, C.c_int64, C.POINTER(C.c_void_p)], S),
            "bucket_plan": ([C.c_int32, P, C.c_int64, P, P, C.c_int32, C.POINTER(C.c_int32)], S),
            "snapshot_shard": ([P, C.c_int32], S),
            "union_compact": ([P, C.c_int32, P, C.c_int64, C.c_int64, P, C.c_int64, P, P], S),
            "union_persist": ([P, C.c_int64, C.POINTER(StepScalars), P, P], S),
            "recover_union": ([P, C.c_int64, P, P, P, C.c_int32, C.POINTER(C.c_int64), P], S),
            "replica_init": ([P, C.c_int64, P, P, P, C.c_int32, P], S),
            "replica_step": ([P, C.c_int64, C.POINTER(StepScalars)], S),
            "replica_persist": ([P], S),
            "replica_wait": ([P, C.POINTER(C.c_int64), C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                              C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_int64)], S),
            "replica_restore": ([P, P, P, P, C.POINTER(C.c_int64), P], S),
            "host_adam_step": ([C.c_int64, P, C.POINTER(AdamConsts), C.POINTER(StepScalars), P, P, P, C.c_int32], S),
            "host_sgd_step": ([C.c_int64, P, C.c_float, P, C.c_int32], S),
            "sync": ([P], S),
            "get_stats": ([P, C.POINTER(Stats)], S),
            "compress_trace": ([P, C.c_int32, C.POINTER(C.c_int32), P, P, P, P], S),
            "prof_enable": ([P, C.c_int32], S),
            "prof_read": ([P, C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)], S),
            "kernel_launches": ([P], C.c_int64),
            "set_graphs": ([P, C.c_int32], S),
            "set_batch_mode": ([P, C.c_int32], S),
            "last_error": ([P], C.c_char_p),
            "nccl_unique_id": ([P], S),
            "derive_step_scalars": ([C.c_int64, C.c_double, C.c_double, C.c_double, C.POINTER(StepScalars)], S),
            "derive_adam_consts": ([C.c_double, C.c_double, C.c_double, C.POINTER(AdamConsts)], S),
            "crc32c": ([P, C.c_size_t], C.c_uint32),
            "chain_scan": ([C.POINTER(Config), C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], S),
            "write_batch_host": ([C.POINTER(Config), C.c_int64, C.c_int32, C.POINTER(StepScalars), P], S),
            "write_full_host": ([C.POINTER(Config), C.c_int64, P, P, P], S),
            "retire_from": ([C.POINTER(Config), C.c_int64, C.c_int32], S),
            "abi_version": ([], C.c_int32),
            "selftest": ([C.c_int32, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)], S),
            "wasted_time": ([C.POINTER(SysParams), C.c_double, C.c_double, C.POINTER(C.c_double)], S),
            "optimal_config": ([C.POINTER(SysParams), C.POINTER(C.c_double), C.POINTER(C.c_double)], S),
            "optimal_config_feasible": ([C.POINTER(SysParams)] + [C.POINTER(C.c_double)] * 4 + [C.POINTER(C.c_int32)], S),
            "config_step": ([C.POINTER(SysParams), C.POINTER(C.c_int64), C.POINTER(C.c_int32)], S),
            "simulate_failures": ([C.POINTER(SysParams), C.c_double, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                   C.POINTER(SimReport)], S),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, "lowdiff_" + name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


EXPORTED = ["create", "destroy", "query", "layer_k", "compress", "residual_materialize", "exchange", "merge", "exchange_update", "peer_alloc", "ipc_open",
            "peer_set", "exchange_peer", "exchange_peer_update", "batch_persist",
            "full_ckpt", "wait_persist", "recover", "replay", "replay_range", "recover_sharded", "snapshot_layer", "snapshot_wait", "snapshot_shard", "bucket_plan", "union_compact", "union_persist", "recover_union",
            "replica_init",
            "replica_step", "replica_persist", "replica_wait", "replica_restore", "host_adam_step", "host_sgd_step",
            "sync", "get_stats", "compress_trace",
            "prof_enable", "prof_read", "kernel_launches", "set_graphs", "set_batch_mode", "last_error", "nccl_unique_id",
            "derive_step_scalars", "derive_adam_consts", "crc32c", "chain_scan", "write_batch_host", "retire_from",
            "write_full_host", "abi_version", "selftest", "wasted_time", "optimal_config", "optimal_config_feasible", "config_step",
            "simulate_failures"]


def wasted_time(params: dict, f: float, b: float) -> float:
    """Eq. 3 of the paper; params keys N, M, W, S, T, R_F, R_D."""
    out = C.c_double()
    _check("wasted_time", lib().lowdiff_wasted_time(C.byref(SysParams(**params)), f, b, C.byref(out)))
    return out.value


def optimal_config(params: dict):
    """Eq. 5: (f*, b*)."""
    f, b = C.c_double(), C.c_double()
    _check("optimal_config", lib().lowdiff_optimal_config(C.byref(SysParams(**params)), C.byref(f), C.byref(b)))
    return f.value, b.value


def optimal_config_feasible(params: dict):
    """Eq. 5 restricted to f b <= 1: (f, b, clamped, f_unconstrained, b_unconstrained)."""
    f, b, fu, bu, cl = C.c_double(), C.c_double(), C.c_double(), C.c_double(), C.c_int32()
    _check("optimal_config_feasible", lib().lowdiff_optimal_config_feasible(
        C.byref(SysParams(**params)), C.byref(f), C.byref(b), C.byref(fu), C.byref(bu), C.byref(cl)))
    return f.value, b.value, bool(cl.value), fu.value, bu.value


def config_step(params: dict, fcf: int, batch: int):
    """One stepwise adaptation of (full-checkpoint interval, batch size)."""
    f, b = C.c_int64(fcf), C.c_int32(batch)
    _check("config_step", lib().lowdiff_config_step(C.byref(SysParams(**params)), C.byref(f), C.byref(b)))
    return f.value, b.value


def simulate_failures(params: dict, f: float, b: float, sw_fraction: float = 0.0, R_S: float = 0.0,
                      seed: int = 0) -> dict:
    """Failure-injection simulator: the wasted-time ledger of one failure trace."""
    out = SimReport()
    _check("simulate_failures", lib().lowdiff_simulate_failures(C.byref(SysParams(**params)), f, b, sw_fraction, R_S,
                                                                seed, C.byref(out)))
    return {k: getattr(out, k) for k, _ in SimReport._fields_}


def selftest(which: int, n: int = 0, seed: int = 0):
    """(mismatches, first_bad) of the device IEEE helpers vs the CUDA intrinsics (needs a GPU)."""
    bad, first = C.c_uint64(), C.c_uint64()
    _check("selftest", lib().lowdiff_selftest(which, n, seed, C.byref(bad), C.byref(first)))
    return bad.value, first.value


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        assert t.is_contiguous(), "tensors must be contiguous"
        return C.c_void_p(t.data_ptr())
    return C.c_void_p(int(t))


def _device_view(addr, n):
    """An int32 CUDA tensor of n elements viewing library-owned device memory at addr (not owned)."""
    class _Arr:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (addr, False), "version": 3,
                                    "strides": None}
    return torch.as_tensor(_Arr(), device="cuda")


def _stream(s):
    if s is None:
        s = torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream if hasattr(s, "cuda_stream") else int(s))


def derive_step_scalars(t: int, lr: float, beta1: float = 0.9, beta2: float = 0.999) -> StepScalars:
    out = StepScalars()
    _check("derive_step_scalars", lib().lowdiff_derive_step_scalars(t, lr, beta1, beta2, C.byref(out)))
    return out


def derive_adam_consts(beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8) -> AdamConsts:
    out = AdamConsts()
    _check("derive_adam_consts", lib().lowdiff_derive_adam_consts(beta1, beta2, eps, C.byref(out)))
    return out


def crc32c(data: bytes) -> int:
    buf = C.create_string_buffer(data, len(data))
    return int(lib().lowdiff_crc32c(buf, len(data)))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check("nccl_unique_id", lib().lowdiff_nccl_unique_id(buf))
    return buf.raw


def _check(fn, code, ctx=None):
    if code != OK:
        msg = ""
        if ctx is not None:
            m = lib().lowdiff_last_error(ctx)
            msg = m.decode() if m else ""
        raise LowDiffError(fn, code, msg)


@dataclass
class Options:
    density_ppm: int = 10000
    error_feedback: bool = True
    mean: bool = True
    rank: int = 0
    world: int = 1
    nccl_id: bytes | None = None
    device: int = 0
    ckpt_dir: str | None = None
    batch_size: int = 1
    ring_slots: int = 0
    write_files: bool = True
    fsync: bool = False
    optim: int = ADAM
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8


def make_config(sizes, o: Options):
    numel = (C.c_int64 * len(sizes))(*[int(n) for n in sizes])
    idbuf = C.create_string_buffer(o.nccl_id, 128) if o.nccl_id is not None else None
    cfg = Config(len(sizes), numel, o.density_ppm, int(o.error_feedback), int(o.mean), o.rank, o.world,
                 C.cast(idbuf, C.c_void_p) if idbuf is not None else None, o.device,
                 o.ckpt_dir.encode() if o.ckpt_dir else None, o.batch_size, o.ring_slots, int(o.write_files),
                 int(o.fsync), o.optim, derive_adam_consts(o.beta1, o.beta2, o.eps))
    cfg._keep = (numel, idbuf)   # keep the buffers alive with the struct
    return cfg


class Context:
    """One lowdiff_ctx (one per process and GPU)."""

    def __init__(self, sizes, opts: Options | None = None, **kw):
        o = opts or Options(**kw)
        self.opts = o
        self.sizes = [int(n) for n in sizes]
        self._cfg = make_config(self.sizes, o)
        h = C.c_void_p()
        _check("create", lib().lowdiff_create(C.byref(self._cfg), C.byref(h)))
        self._h = h
        psi, K = C.c_int64(), C.c_int64()
        _check("query", lib().lowdiff_query(h, C.byref(psi), C.byref(K)), h)
        self.psi, self.K = psi.value, K.value

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            h, self._h = self._h, None
            _check("destroy", lib().lowdiff_destroy(h))

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _c(self, fn, code):
        _check(fn, code, self._h)

    # -- the five calls
    def compress(self, grad, residual, send, stream=None):
        self._c("compress", lib().lowdiff_compress(self._h, _ptr(grad), _ptr(residual), _ptr(send), _stream(stream)))

    def residual_materialize(self, residual, stream=None):
        self._c("residual_materialize", lib().lowdiff_residual_materialize(self._h, _ptr(residual), _stream(stream)))

    def exchange(self, send, gathered, dense_out, stream=None):
        self._c("exchange", lib().lowdiff_exchange(self._h, _ptr(send), _ptr(gathered), _ptr(dense_out),
                                                   _stream(stream)))

    def merge(self, world, gathered, dense_out, stream=None):
        self._c("merge", lib().lowdiff_merge(self._h, world, _ptr(gathered), _ptr(dense_out), _stream(stream)))

    def exchange_update(self, send, gathered, scalars: StepScalars, p, m=None, v=None, stream=None):
        self._c("exchange_update", lib().lowdiff_exchange_update(self._h, _ptr(send), _ptr(gathered), C.byref(scalars),
                                                                 _ptr(p), _ptr(m), _ptr(v), _stream(stream)))

    # -- peer-memory exchange (NEXT-1)
    def peer_alloc(self, n_slots=2, handles=True):
        """Allocates the library's send slots; returns (slot tensors u32[2K] as int32 views, handle bytes)."""
        ptrs = (C.c_void_p * n_slots)()
        hbuf = C.create_string_buffer(64 * (n_slots + 1)) if handles else None
        flags = C.c_void_p()
        self._c("peer_alloc", lib().lowdiff_peer_alloc(self._h, n_slots, ptrs, C.byref(flags), hbuf))
        self.peer_n = n_slots
        self.peer_ptrs = [int(p) for p in ptrs]
        self.peer_flags_ptr = int(flags.value)
        return [_device_view(p, 2 * self.K) for p in self.peer_ptrs], (hbuf.raw if handles else None)

    def ipc_open(self, handle: bytes) -> int:
        out = C.c_void_p()
        self._c("ipc_open", lib().lowdiff_ipc_open(self._h, C.create_string_buffer(handle, 64), C.byref(out)))
        return out.value

    def peer_set(self, table):
        """table: world x (n_slots + 1) device addresses (rank order; each rank's slots then flags)."""
        flat = [int(x) for row in table for x in row]
        arr = (C.c_void_p * len(flat))(*flat)
        self._c("peer_set", lib().lowdiff_peer_set(self._h, arr))

    def peer_setup(self, n_slots=2, group=None):
        """Multi-process setup over torch.distributed: allocate, share IPC handles, map the peers'."""
        import torch.distributed as dist
        slots, h = self.peer_alloc(n_slots, handles=True)
        world, rank = self.opts.world, self.opts.rank
        allh = [None] * world
        dist.all_gather_object(allh, h, group=group)
        table = []
        for q in range(world):
            if q == rank:
                table.append(self.peer_ptrs + [self.peer_flags_ptr])
            else:
                table.append([self.ipc_open(allh[q][64 * i:64 * (i + 1)]) for i in range(n_slots + 1)])
        self.peer_set(table)
        return slots

    def exchange_peer(self, slot, dense_out, stream=None):
        self._c("exchange_peer", lib().lowdiff_exchange_peer(self._h, slot, _ptr(dense_out), _stream(stream)))

    def exchange_peer_update(self, slot, scalars: StepScalars, p, m=None, v=None, stream=None):
        self._c("exchange_peer_update", lib().lowdiff_exchange_peer_update(self._h, slot, C.byref(scalars), _ptr(p),
                                                                           _ptr(m), _ptr(v), _stream(stream)))

    def batch_persist(self, iteration, scalars: StepScalars, send, stream=None):
        self._c("batch_persist", lib().lowdiff_batch_persist(self._h, iteration, C.byref(scalars), _ptr(send),
                                                             _stream(stream)))

    def wait_persist(self, stream=None):
        self._c("wait_persist", lib().lowdiff_wait_persist(self._h, _stream(stream)))

    def full_ckpt(self, iteration, p, m=None, v=None, stream=None):
        self._c("full_ckpt", lib().lowdiff_full_ckpt(self._h, iteration, _ptr(p), _ptr(m), _ptr(v), _stream(stream)))

    def recover(self, p, m=None, v=None, target=-1, stream=None) -> int:
        rec = C.c_int64(-1)
        self._c("recover", lib().lowdiff_recover(self._h, target, _ptr(p), _ptr(m), _ptr(v), C.byref(rec),
                                                 _stream(stream)))
        return rec.value

    def replay(self, optim, world, n_steps, diffs, scalars, p, m=None, v=None, stream=None):
        arr = (StepScalars * max(1, n_steps))(*scalars)
        self._c("replay", lib().lowdiff_replay(self._h, optim, world, n_steps, _ptr(diffs), arr, _ptr(p), _ptr(m),
                                               _ptr(v), _stream(stream)))
        self._keep_scalars = arr

    def replay_range(self, optim, world, n_steps, diffs, scalars, begin, end, p, m=None, v=None, stream=None):
        """p, m, v: device float32 tensors of end - begin elements (the range only)."""
        arr = (StepScalars * max(1, n_steps))(*scalars)
        self._c("replay_range", lib().lowdiff_replay_range(self._h, optim, world, n_steps, _ptr(diffs), arr, begin, end,
                                                           _ptr(p), _ptr(m), _ptr(v), _stream(stream)))
        self._keep_scalars = arr

    def recover_sharded(self, p, m=None, v=None, target=-1, gather=True, stream=None) -> int:
        it = C.c_int64()
        self._c("recover_sharded", lib().lowdiff_recover_sharded(self._h, target, _ptr(p), _ptr(m), _ptr(v),
                                                                 int(bool(gather)), C.byref(it), _stream(stream)))
        return it.value

    def union_compact(self, world, gathered, begin, end, out, cap, count_dev, stream=None):
        """C^U_t of [begin, end) into out = idx u32[cap] | val u32[cap]; count in count_dev (u64)."""
        self._c("union_compact", lib().lowdiff_union_compact(self._h, world, _ptr(gathered), begin, end, _ptr(out),
                                                             cap, _ptr(count_dev), _stream(stream)))

    def union_persist(self, iteration, scalars: StepScalars, gathered, stream=None):
        self._c("union_persist", lib().lowdiff_union_persist(self._h, iteration, C.byref(scalars), _ptr(gathered),
                                                             _stream(stream)))

    def recover_union(self, p, m=None, v=None, target=-1, sharded=False, stream=None) -> int:
        rec = C.c_int64()
        self._c("recover_union", lib().lowdiff_recover_union(self._h, target, _ptr(p), _ptr(m), _ptr(v),
                                                             int(bool(sharded)), C.byref(rec), _stream(stream)))
        return rec.value

    def snapshot_layer(self, iteration, first_layer, n_layers, grad_bucket, stream=None):
        self._c("snapshot_layer", lib().lowdiff_snapshot_layer(self._h, iteration, first_layer, n_layers,
                                                               _ptr(grad_bucket), _stream(stream)))

    def snapshot_shard(self, on=True):
        """Copy only this rank's 1/world shard of each snapshotted bucket."""
        self._c("snapshot_shard", lib().lowdiff_snapshot_shard(self._h, int(bool(on))))

    def snapshot_wait(self, iteration):
        """Returns a CPU float32 tensor viewing the pinned snapshot buffer (valid until iteration + 2)."""
        p = C.c_void_p()
        self._c("snapshot_wait", lib().lowdiff_snapshot_wait(self._h, iteration, C.byref(p)))
        arr = (C.c_float * self.psi).from_address(p.value)
        return torch.frombuffer(arr, dtype=torch.float32)

    # -- LowDiff+ CPU replica (Alg. 2 l.11-13)
    def replica_init(self, iteration, p, m=None, v=None, threads=None, stream=None):
        threads = threads or max(1, min(32, (os.cpu_count() or 1)))
        self._c("replica_init", lib().lowdiff_replica_init(self._h, iteration, _ptr(p), _ptr(m), _ptr(v), threads,
                                                           _stream(stream)))

    def replica_step(self, iteration, scalars: StepScalars):
        self._c("replica_step", lib().lowdiff_replica_step(self._h, iteration, C.byref(scalars)))

    def replica_persist(self):
        self._c("replica_persist", lib().lowdiff_replica_persist(self._h))

    def replica_wait(self):
        """Drains the replica; returns (iteration, p, m, v, shard_begin, shard_end), p/m/v CPU float32
        tensors viewing the pinned replica shard (valid until more replica work is queued)."""
        it, sb, se = C.c_int64(), C.c_int64(), C.c_int64()
        ptr = [C.c_void_p() for _ in range(3)]
        self._c("replica_wait", lib().lowdiff_replica_wait(self._h, C.byref(it), *[C.byref(x) for x in ptr],
                                                           C.byref(sb), C.byref(se)))
        n = se.value - sb.value
        views = [torch.frombuffer((C.c_float * max(1, n)).from_address(x.value), dtype=torch.float32)[:n]
                 for x in ptr]
        return (it.value, *views, sb.value, se.value)

    def replica_restore(self, p, m=None, v=None, stream=None) -> int:
        it = C.c_int64()
        self._c("replica_restore", lib().lowdiff_replica_restore(self._h, _ptr(p), _ptr(m), _ptr(v), C.byref(it),
                                                                 _stream(stream)))
        return it.value

    def sync(self):
        self._c("sync", lib().lowdiff_sync(self._h))

    # -- introspection
    def layer_k(self, layer):
        k, koff = C.c_int64(), C.c_int64()
        self._c("layer_k", lib().lowdiff_layer_k(self._h, layer, C.byref(k), C.byref(koff)))
        return k.value, koff.value

    def stats(self) -> dict:
        s = Stats()
        self._c("get_stats", lib().lowdiff_get_stats(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in Stats._fields_}

    def compress_trace(self):
        """Per large layer of the last compress: (layer ids, level 0/1/2, candidates, threshold key)."""
        import numpy as np
        n = C.c_int32()
        self._c("compress_trace", lib().lowdiff_compress_trace(self._h, 0, C.byref(n), None, None, None, None))
        L, lev = np.zeros(n.value, np.int32), np.zeros(n.value, np.int32)
        cand, thr = np.zeros(n.value, np.uint32), np.zeros(n.value, np.uint32)
        self._c("compress_trace", lib().lowdiff_compress_trace(self._h, n.value, C.byref(n), *[a.ctypes.data_as(C.c_void_p)
                                                                                             for a in (L, lev, cand, thr)]))
        return L, lev, cand, thr

    def set_graphs(self, on=True):
        """Replay compress / merge as captured CUDA graphs (fewer launch gaps for small models)."""
        self._c("set_graphs", lib().lowdiff_set_graphs(self._h, int(bool(on))))

    def set_batch_mode(self, mode):
        """BATCH_RECORD (exact) or BATCH_ACCUMULATED (the paper's tensor-addition batching of the
        union dictionaries; one replay step per batch, inexact for b > 1) -- include/lowdiff.h."""
        self._c("set_batch_mode", lib().lowdiff_set_batch_mode(self._h, int(mode)))

    def prof_enable(self, on=True):
        self._c("prof_enable", lib().lowdiff_prof_enable(self._h, int(on)))

    def prof_read(self, name=""):
        ms, n = C.c_double(), C.c_int64()
        self._c("prof_read", lib().lowdiff_prof_read(self._h, name.encode(), C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def kernel_launches(self) -> int:
        return int(lib().lowdiff_kernel_launches(self._h))


def chain_scan(sizes, opts: Options, target=-1):
    cfg = make_config(sizes, opts)
    f, l = C.c_int64(), C.c_int64()
    _check("chain_scan", lib().lowdiff_chain_scan(C.byref(cfg), target, C.byref(f), C.byref(l)))
    return f.value, l.value


def write_batch_host(sizes, opts: Options, first_iter, scalars, blocks):
    """blocks: numpy/torch uint32 array [n_iters, 2K] on the host."""
    import numpy as np
    cfg = make_config(sizes, opts)
    b = np.ascontiguousarray(np.asarray(blocks, dtype=np.uint32))
    arr = (StepScalars * len(scalars))(*scalars)
    _check("write_batch_host", lib().lowdiff_write_batch_host(C.byref(cfg), first_iter, len(scalars), arr,
                                                              b.ctypes.data_as(C.c_void_p)))


def bucket_plan(sizes, min_bytes=4 << 20):
    """LowDiff+ snapshot buckets in backward order: [(first_layer, n_layers), ...]."""
    n = len(sizes)
    numel = (C.c_int64 * n)(*sizes)
    first, count, nb = (C.c_int32 * n)(), (C.c_int32 * n)(), C.c_int32()
    _check("bucket_plan", lib().lowdiff_bucket_plan(n, numel, min_bytes, first, count, n, C.byref(nb)))
    return [(first[i], count[i]) for i in range(nb.value)]


def host_adam_step(G, consts: AdamConsts, scalars: StepScalars, p, m, v, threads=1):
    """The replica's host Adam on numpy float32 arrays (p, m, v updated in place)."""
    import numpy as np
    for a in (p, m, v):
        assert a.dtype == np.float32 and a.flags.c_contiguous
    g = np.ascontiguousarray(G, dtype=np.float32)
    assert g.size == p.size == m.size == v.size
    _check("host_adam_step", lib().lowdiff_host_adam_step(p.size, g.ctypes.data_as(C.c_void_p), C.byref(consts),
                                                          C.byref(scalars), *[a.ctypes.data_as(C.c_void_p)
                                                                              for a in (p, m, v)], threads))


def host_sgd_step(G, lr, p, threads=1):
    import numpy as np
    assert p.dtype == np.float32 and p.flags.c_contiguous
    g = np.ascontiguousarray(G, dtype=np.float32)
    assert g.size == p.size
    _check("host_sgd_step", lib().lowdiff_host_sgd_step(p.size, g.ctypes.data_as(C.c_void_p), lr,
                                                        p.ctypes.data_as(C.c_void_p), threads))


def retire_from(sizes, opts: Options, iteration, kinds=7):
    """Remove / truncate opts.rank's files holding iterations >= iteration (restart hygiene)."""
    cfg = make_config(sizes, opts)
    _check("retire_from", lib().lowdiff_retire_from(C.byref(cfg), iteration, kinds))


def write_full_host(sizes, opts: Options, iteration, p, m=None, v=None):
    import numpy as np
    cfg = make_config(sizes, opts)
    arrs = [None if a is None else np.ascontiguousarray(np.asarray(a, dtype=np.float32)) for a in (p, m, v)]
    ptrs = [None if a is None else a.ctypes.data_as(C.c_void_p) for a in arrs]
    _check("write_full_host", lib().lowdiff_write_full_host(C.byref(cfg), iteration, *ptrs))
