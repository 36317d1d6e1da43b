"""Python binding of the Polar Express B200 C-ABI library (include/pe.h).

Argument marshalling only: every step of the path runs in libpe.so's CUDA
kernels (sm_100a).  There is no CPU or PyTorch fallback -- if the library is
missing or the device is not a B200, calls raise.

Names follow the C ABI: ``pe_coeffs``, ``pe_coeffs_ex``, ``pe_polar``,
``pe_polar_host``, ``pe_shard_plan``, ``pe_flops``; a ``Context`` wraps
``pe_create`` / ``pe_destroy`` / ``pe_set_coeffs`` / ``pe_reserve``.
"""
from __future__ import annotations

import ctypes
import os

__all__ = [
    "PE_BF16", "PE_FP32", "PE_SAFETY_ALL", "PE_SAFETY_NOT_FINAL", "PE_NO_RECENTER",
    "PeError", "lib", "pe_coeffs", "pe_coeffs_ex", "pe_shard_plan", "pe_shard_buckets", "pe_flops",
    "pe_nccl_unique_id",
    "Context", "pe_polar", "pe_polar_host", "MuonPE", "EXPORTED_SYMBOLS",
]

PE_BF16 = 0
PE_FP32 = 1
PE_SAFETY_ALL = 1
PE_SAFETY_NOT_FINAL = 2
PE_NO_RECENTER = 4

_STATUS = {0: "PE_OK", 1: "PE_ERR_INVALID_ARG", 2: "PE_ERR_UNSUPPORTED", 3: "PE_ERR_NO_CONVERGENCE",
           4: "PE_ERR_CUDA", 5: "PE_ERR_NCCL", 6: "PE_ERR_WORKSPACE",
           7: "PE_ERR_NONFINITE"}

EXPORTED_SYMBOLS = [
    "pe_status_string", "pe_version", "pe_last_error_message", "pe_coeffs", "pe_coeffs_ex",
    "pe_create", "pe_destroy", "pe_set_coeffs", "pe_reserve", "pe_polar", "pe_polar_host",
    "pe_last_launch_count", "pe_shard_plan", "pe_flops", "pe_profile_enable", "pe_profile_read",
    "pe_muon_step", "pe_polar_split", "pe_shard_buckets", "pe_nccl_unique_id", "pe_attach_comm",
    "pe_comm_info", "pe_polar_sharded", "pe_polar_ex", "pe_set_spectrum_init",
    "pe_set_spectrum_init_ex", "pe_attach_exchange", "pe_shard_nbuckets", "pe_shard_layout",
    "pe_set_rect_iteration", "pe_sharded_exchange", "pe_count_nonfinite", "pe_set_debug",
    "pe_set_small_planes", "pe_split_slot_bytes", "pe_polar_split_peers",
]
PROFILE_KINDS = ["norm", "scale", "gram", "poly", "update", "transpose_back", "fused", "small"]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PE_LIB_OVERRIDE") or os.path.join(_HERE, "libpe.so")   # override: A/B experiments only


class PeError(RuntimeError):
    def __init__(self, status, where, detail=""):
        self.status = status
        super().__init__(f"{where}: {_STATUS.get(status, status)}" + (f" ({detail})" if detail else ""))


_lib = None


def lib():
    """Load libpe.so (building it first if it is absent and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _build
        _build.build()
    L = ctypes.CDLL(LIB_PATH)
    P, I, D, I64P = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_int64)
    DP = ctypes.POINTER(ctypes.c_double)
    sig = {
        "pe_status_string": (ctypes.c_char_p, [I]),
        "pe_version": (ctypes.c_char_p, []),
        "pe_last_error_message": (ctypes.c_char_p, []),
        "pe_coeffs": (I, [D, I, I, D, DP]),
        "pe_coeffs_ex": (I, [D, I, I, D, D, I, DP, DP]),
        "pe_create": (I, [ctypes.POINTER(P), I]),
        "pe_destroy": (I, [P]),
        "pe_set_coeffs": (I, [P, DP, I, I]),
        "pe_reserve": (I, [P, I64P, I, I]),
        "pe_polar": (I, [P, ctypes.POINTER(P), ctypes.POINTER(P), I64P, I, I, I, P]),
        "pe_polar_host": (I, [P, ctypes.POINTER(P), ctypes.POINTER(P), I64P, I, I, I, P]),
        "pe_polar_ex": (I, [P, ctypes.POINTER(P), ctypes.POINTER(P), I64P, I, I, I, I, I, P]),
        "pe_set_spectrum_init": (I, [P, I]),
        "pe_set_spectrum_init_ex": (I, [P, I, D]),
        "pe_set_rect_iteration": (I, [P, I, D, D]),
        "pe_sharded_exchange": (I, [P, ctypes.POINTER(P), I64P, I, I, P]),
        "pe_count_nonfinite": (I, [P, ctypes.POINTER(P), I64P, I, I, ctypes.POINTER(ctypes.c_int64), P]),
        "pe_set_debug": (I, [P, I]),
        "pe_set_small_planes": (I, [P, I]),
        "pe_split_slot_bytes": (I, [ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]),
        "pe_polar_split_peers": (I, [P, P, P, ctypes.c_int64, ctypes.c_int64, I, ctypes.POINTER(P), I, I,
                                     BARRIER_FN, P, P]),
        "pe_last_launch_count": (I, [P, ctypes.POINTER(I)]),
        "pe_shard_plan": (I, [I64P, I, I, ctypes.POINTER(I)]),
        "pe_flops": (I, [I64P, I, I, I, DP]),
        "pe_profile_enable": (I, [P, I]),
        "pe_profile_read": (I, [P, DP, ctypes.POINTER(I), I]),
        "pe_muon_step": (I, [P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P), I64P, I, D, D, I, P]),
        "pe_polar_split": (I, [P, P, P, ctypes.c_int64, ctypes.c_int64, I, ALLREDUCE_FN, P, P]),
        "pe_shard_buckets": (I, [I64P, I, I, ctypes.POINTER(I)]),
        "pe_nccl_unique_id": (I, [ctypes.c_char_p]),
        "pe_attach_comm": (I, [P, ctypes.c_char_p, I, I]),
        "pe_comm_info": (I, [P, ctypes.POINTER(I), ctypes.POINTER(I)]),
        "pe_polar_sharded": (I, [P, ctypes.POINTER(P), ctypes.POINTER(P), I64P, I, I, I, P]),
        "pe_attach_exchange": (I, [P, I, I, EXCHANGE_FN, P]),
        "pe_shard_nbuckets": (I, [I64P, I, I, ctypes.POINTER(I)]),
        "pe_shard_layout": (I, [I64P, I, I, I, I64P, I64P, I64P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


# pe_allreduce_fn (include/pe.h): (buf, count, dtype 0 fp32 / 1 fp64, user, stream) -> pe_status
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                ctypes.c_void_p)


# pe_exchange_fn (include/pe.h): (op, buf, bytes, root, user, stream) -> pe_status
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                               ctypes.c_void_p, ctypes.c_void_p)
PE_EXCHANGE_ALLGATHER, PE_EXCHANGE_BROADCAST = 0, 1
# pe_barrier_fn (include/pe.h): (user, stream) -> pe_status
BARRIER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p)
PE_DEBUG_CHECK_FINITE = 1


class _DevBuf:
    """A raw device buffer seen through __cuda_array_interface__ (zero copy)."""

    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2}


def _check(status, where):
    if status != 0:
        detail = lib().pe_last_error_message()
        raise PeError(status, where, detail.decode() if detail else "")


def _shapes_arr(shapes):
    flat = []
    for r, c in shapes:
        flat += [int(r), int(c)]
    return (ctypes.c_int64 * max(1, len(flat)))(*flat)


def pe_coeffs(ell=1e-3, degree=5, T=8, safety=1.01):
    """Offline stage (pe.h pe_coeffs): list of T tuples (a, b[, c])."""
    nq = (degree + 1) // 2
    buf = (ctypes.c_double * (max(T, 1) * nq))()
    _check(lib().pe_coeffs(float(ell), int(degree), int(T), float(safety), buf), "pe_coeffs")
    return [tuple(buf[t * nq:(t + 1) * nq]) for t in range(T)]


def pe_coeffs_ex(ell=1e-3, degree=5, T=8, safety=1.01, cushion=-1.0, flags=0):
    """pe.h pe_coeffs_ex: (tuples, ell_trace[T+1])."""
    nq = (degree + 1) // 2
    buf = (ctypes.c_double * (max(T, 1) * nq))()
    tr = (ctypes.c_double * (max(T, 1) + 1))()
    _check(lib().pe_coeffs_ex(float(ell), int(degree), int(T), float(safety), float(cushion), int(flags),
                              buf, tr), "pe_coeffs_ex")
    return [tuple(buf[t * nq:(t + 1) * nq]) for t in range(T)], list(tr[:T + 1])


def pe_shard_plan(shapes, world):
    """pe.h pe_shard_plan: owner rank per matrix (deterministic LPT)."""
    n = len(shapes)
    own = (ctypes.c_int * max(n, 1))()
    _check(lib().pe_shard_plan(_shapes_arr(shapes), n, int(world), own), "pe_shard_plan")
    return list(own[:n])


def pe_shard_buckets(shapes, nbuckets):
    """First matrix index of each of `nbuckets` cost-balanced consecutive
    buckets, plus len(shapes) at the end (pe_polar_sharded's exchange order)."""
    n = len(shapes)
    beg = (ctypes.c_int * (nbuckets + 1))()
    _check(lib().pe_shard_buckets(_shapes_arr(shapes), n, int(nbuckets), beg), "pe_shard_buckets")
    return list(beg)


def pe_shard_nbuckets(shapes, world):
    """pe.h pe_shard_nbuckets: pe_polar_sharded's bucket count for this set."""
    n = ctypes.c_int()
    _check(lib().pe_shard_nbuckets(_shapes_arr(shapes), len(shapes), int(world), ctypes.byref(n)),
           "pe_shard_nbuckets")
    return n.value


def pe_shard_layout(shapes, world, dtype=PE_BF16, chunks=False):
    """pe.h pe_shard_layout: (byte offset of every matrix, total bytes) of the
    flat output buffer that makes pe_polar_sharded's exchange one in-place
    all-gather per bucket; with chunks=True also the per-rank chunk bytes of
    every bucket: (offsets, chunk_bytes, total)."""
    n = len(shapes)
    offs = (ctypes.c_int64 * max(n, 1))()
    nb = pe_shard_nbuckets(shapes, world)
    ch = (ctypes.c_int64 * max(nb, 1))()
    tot = ctypes.c_int64()
    _check(lib().pe_shard_layout(_shapes_arr(shapes), n, int(world), int(dtype), offs, ch, ctypes.byref(tot)),
           "pe_shard_layout")
    if chunks:
        return list(offs[:n]), list(ch[:nb]), tot.value
    return list(offs[:n]), tot.value


def pe_split_slot_bytes(rows, cols):
    """pe.h pe_split_slot_bytes: bytes of one rank's slot for pe_polar_split_peers."""
    out = ctypes.c_int64()
    _check(lib().pe_split_slot_bytes(int(rows), int(cols), ctypes.byref(out)), "pe_split_slot_bytes")
    return out.value


def pe_nccl_unique_id():
    """A fresh 128-byte ncclUniqueId (make it on one rank, share it out of band)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().pe_nccl_unique_id(buf), "pe_nccl_unique_id")
    return buf.raw


def pe_flops(shapes, iters, degree=5):
    """pe.h pe_flops: algorithmic flops of one call."""
    out = ctypes.c_double()
    _check(lib().pe_flops(_shapes_arr(shapes), len(shapes), int(iters), int(degree), ctypes.byref(out)),
           "pe_flops")
    return out.value


def _dtype_code(t):
    import torch
    if t.dtype == torch.bfloat16:
        return PE_BF16
    if t.dtype == torch.float32:
        return PE_FP32
    raise TypeError(f"unsupported dtype {t.dtype}")


class Context:
    """One pe_ctx on a CUDA device."""

    def __init__(self, device=0):
        self._h = ctypes.c_void_p()
        _check(lib().pe_create(ctypes.byref(self._h), int(device)), "pe_create")
        self.device = int(device)

    def close(self):
        if self._h:
            lib().pe_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_coeffs(self, tuples):
        deg = 2 * len(tuples[0]) - 1
        flat = [float(v) for t in tuples for v in t]
        arr = (ctypes.c_double * len(flat))(*flat)
        _check(lib().pe_set_coeffs(self._h, arr, len(tuples), deg), "pe_set_coeffs")

    def set_spectrum_init(self, power_iters, margin=None):
        """pe_set_spectrum_init: App. G's spectrum-aware first step with
        `power_iters` power-method steps (0 = off); `margin` (reading R17,
        default 2^-7 = pe_set_spectrum_init) goes to pe_set_spectrum_init_ex,
        0 = eq. (init_poly) exactly."""
        if margin is None:
            _check(lib().pe_set_spectrum_init(self._h, int(power_iters)), "pe_set_spectrum_init")
        else:
            _check(lib().pe_set_spectrum_init_ex(self._h, int(power_iters), float(margin)),
                   "pe_set_spectrum_init_ex")

    def count_nonfinite(self, tensors, stream=None):
        """pe_count_nonfinite: NaN / Inf elements over CUDA tensors of one dtype."""
        import torch
        n = len(tensors)
        ptrs = (ctypes.c_void_p * max(n, 1))(*[t.data_ptr() for t in tensors])
        out = ctypes.c_int64()
        if stream is None:
            stream = torch.cuda.current_stream(tensors[0].device)
        _check(lib().pe_count_nonfinite(self._h, ptrs, _shapes_arr([tuple(t.shape) for t in tensors]), n,
                                        _dtype_code(tensors[0]), ctypes.byref(out),
                                        ctypes.c_void_p(stream.cuda_stream)), "pe_count_nonfinite")
        return out.value

    def set_small_planes(self, planes):
        """pe_set_small_planes: 2 (default) keeps A and B of the bf16 small
        path as two bf16 planes (reading R8p); 1 = R8, bit-identical to the
        large path."""
        _check(lib().pe_set_small_planes(self._h, int(planes)), "pe_set_small_planes")

    def set_debug(self, flags):
        """pe_set_debug (PE_DEBUG_CHECK_FINITE = 1)."""
        _check(lib().pe_set_debug(self._h, int(flags)), "pe_set_debug")

    def set_rect_iteration(self, restart, min_aspect=0.0, shift=1e-3):
        """pe_set_rect_iteration: App. H's Alg. 4 for matrices with aspect
        ratio above `min_aspect` (<= 0: the paper's 1.5 T / (T - 1)),
        restarted every `restart` iterations (0 = off), Y shifted by `shift` I
        in the first application."""
        _check(lib().pe_set_rect_iteration(self._h, int(restart), float(min_aspect), float(shift)),
               "pe_set_rect_iteration")

    def reserve(self, shapes, dtype=PE_BF16):
        _check(lib().pe_reserve(self._h, _shapes_arr(shapes), len(shapes), int(dtype)), "pe_reserve")

    def last_launch_count(self):
        n = ctypes.c_int()
        _check(lib().pe_last_launch_count(self._h, ctypes.byref(n)), "pe_last_launch_count")
        return n.value

    def profile_enable(self, on=True):
        _check(lib().pe_profile_enable(self._h, int(bool(on))), "pe_profile_enable")

    def profile_read(self):
        """{kind: (total_ms, launches)} accumulated since the last read."""
        k = len(PROFILE_KINDS)
        ms = (ctypes.c_double * k)()
        cnt = (ctypes.c_int * k)()
        _check(lib().pe_profile_read(self._h, ms, cnt, k), "pe_profile_read")
        return {PROFILE_KINDS[i]: (ms[i], cnt[i]) for i in range(k)}

    def polar(self, inputs, outputs=None, iters=5, stream=None):
        """pe_polar on device tensors (2-D, contiguous, same dtype: bf16 or fp32).
        ``outputs`` defaults to new tensors; pass ``inputs`` for in-place."""
        import torch
        if len(inputs) == 0:
            _check(lib().pe_polar(self._h, None, None, None, 0, int(iters), PE_BF16, None), "pe_polar")
            return []
        dt = _dtype_code(inputs[0])
        if outputs is None:
            outputs = [torch.empty_like(x) for x in inputs]
        for x, y in zip(inputs, outputs):
            if x.dim() != 2 or not x.is_contiguous() or not y.is_contiguous() or x.shape != y.shape:
                raise ValueError("pe_polar takes contiguous 2-D tensors of matching shapes")
            if _dtype_code(x) != dt or _dtype_code(y) != dt or not x.is_cuda or not y.is_cuda:
                raise ValueError("pe_polar takes CUDA tensors of one dtype")
        n = len(inputs)
        ins = (ctypes.c_void_p * n)(*[x.data_ptr() for x in inputs])
        outs = (ctypes.c_void_p * n)(*[y.data_ptr() for y in outputs])
        shp = _shapes_arr([tuple(x.shape) for x in inputs])
        if stream is None:
            stream = torch.cuda.current_stream(inputs[0].device)
        _check(lib().pe_polar(self._h, ins, outs, shp, n, int(iters), dt, ctypes.c_void_p(stream.cuda_stream)),
               "pe_polar")
        return outputs

    def polar_ex(self, inputs, outputs, iters=5, compute=PE_BF16, stream=None):
        """pe_polar_ex: the element types of ``inputs`` and ``outputs`` (bf16 or
        fp32 CUDA tensors, each list of one type) may differ from the
        arithmetic ``compute`` (PE_BF16: fp32 momentum in, bf16 iteration,
        bf16 or fp32 out -- Listing 2's X = G.bfloat16())."""
        import torch
        n = len(inputs)
        if len(outputs) != n:
            raise ValueError("polar_ex takes equally long input / output lists")
        if n == 0:
            return outputs
        di, do = _dtype_code(inputs[0]), _dtype_code(outputs[0])
        for x, y in zip(inputs, outputs):
            if x.dim() != 2 or not x.is_contiguous() or not y.is_contiguous() or x.shape != y.shape:
                raise ValueError("pe_polar_ex takes contiguous 2-D tensors of matching shapes")
            if _dtype_code(x) != di or _dtype_code(y) != do or not x.is_cuda or not y.is_cuda:
                raise ValueError("pe_polar_ex takes CUDA tensors, one dtype per list")
        ins = (ctypes.c_void_p * n)(*[x.data_ptr() for x in inputs])
        outs = (ctypes.c_void_p * n)(*[y.data_ptr() for y in outputs])
        shp = _shapes_arr([tuple(x.shape) for x in inputs])
        if stream is None:
            stream = torch.cuda.current_stream(inputs[0].device)
        _check(lib().pe_polar_ex(self._h, ins, outs, shp, n, int(iters), di, do, int(compute),
                                 ctypes.c_void_p(stream.cuda_stream)), "pe_polar_ex")
        return outputs

    def muon_step(self, weights, momenta, grads, beta=0.9, lr=0.02, iters=5, stream=None):
        """pe_muon_step on bf16 CUDA tensors: momenta <- beta*momenta +
        (1-beta)*grads, weights <- weights - lr * polar(momenta); in place."""
        import torch
        n = len(weights)
        if not (len(momenta) == n and len(grads) == n):
            raise ValueError("muon_step takes equally long weight / momentum / gradient lists")
        for w, m, g in zip(weights, momenta, grads):
            for t in (w, m, g):
                if t.dim() != 2 or not t.is_contiguous() or not t.is_cuda or t.dtype != torch.bfloat16:
                    raise ValueError("muon_step takes contiguous 2-D bf16 CUDA tensors")
            if not (w.shape == m.shape == g.shape):
                raise ValueError("muon_step: weight, momentum and gradient shapes differ")
        W = (ctypes.c_void_p * max(n, 1))(*[t.data_ptr() for t in weights])
        M = (ctypes.c_void_p * max(n, 1))(*[t.data_ptr() for t in momenta])
        G = (ctypes.c_void_p * max(n, 1))(*[t.data_ptr() for t in grads])
        shp = _shapes_arr([tuple(t.shape) for t in weights])
        if stream is None:
            stream = torch.cuda.current_stream(weights[0].device if n else self.device)
        _check(lib().pe_muon_step(self._h, W, M, G, shp, n, float(beta), float(lr), int(iters),
                                  ctypes.c_void_p(stream.cuda_stream)), "pe_muon_step")
        return weights

    def polar_split(self, shard, allreduce=None, out=None, iters=5, stream=None):
        """pe_polar_split: `shard` is this rank's column block M_r (rows x
        cols_r, bf16, cols_r % 8 == 0) of one wide matrix M = [M_0 | M_1 | ...];
        returns the same columns of polar(M).  `allreduce(t)` must sum the CUDA
        tensor `t` in place over all ranks, on the current stream (e.g.
        torch.distributed.all_reduce); None uses the context's own NCCL
        communicator (attach_comm)."""
        import torch
        if shard.dim() != 2 or not shard.is_contiguous() or not shard.is_cuda or shard.dtype != torch.bfloat16:
            raise ValueError("polar_split takes a contiguous 2-D bf16 CUDA tensor")
        if out is None:
            out = torch.empty_like(shard)
        if stream is None:
            stream = torch.cuda.current_stream(shard.device)
        errors = []

        def cb(buf, count, dtype, user, st):
            try:
                t = torch.as_tensor(_DevBuf(buf, count, "<f4" if dtype == 0 else "<f8"), device=shard.device)
                with torch.cuda.stream(torch.cuda.ExternalStream(st or 0, device=shard.device)):
                    allreduce(t)
                return 0
            except Exception as e:          # reported after the call returns
                errors.append(e)
                return 5                    # PE_ERR_NCCL

        fn = ALLREDUCE_FN(cb) if allreduce is not None else ALLREDUCE_FN()
        status = lib().pe_polar_split(self._h, ctypes.c_void_p(shard.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                        int(shard.shape[0]), int(shard.shape[1]), int(iters), fn, None,
                                        ctypes.c_void_p(stream.cuda_stream))
        if errors:
            raise errors[0]
        _check(status, "pe_polar_split")
        return out

    def polar_split_peers(self, shard, slots, rank, barrier, out=None, iters=5, stream=None):
        """pe_polar_split_peers: this rank's column block of one wide matrix;
        `slots` are every rank's slot (device pointers or uint8 CUDA tensors
        of pe_split_slot_bytes bytes, 256-byte aligned, readable by every
        rank), `barrier(stream_handle)` must return once this rank's work on
        the stream is complete and every rank has reached it."""
        import torch
        if shard.dim() != 2 or not shard.is_contiguous() or not shard.is_cuda or shard.dtype != torch.bfloat16:
            raise ValueError("polar_split_peers takes a contiguous 2-D bf16 CUDA tensor")
        if out is None:
            out = torch.empty_like(shard)
        if stream is None:
            stream = torch.cuda.current_stream(shard.device)
        ptrs = [s_.data_ptr() if hasattr(s_, "data_ptr") else int(s_) for s_ in slots]
        arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
        errors = []

        def cb(user, st):
            try:
                barrier(int(st or 0))
                return 0
            except Exception as e:          # reported after the call returns
                errors.append(e)
                return 5
        fn = BARRIER_FN(cb)
        status = lib().pe_polar_split_peers(self._h, ctypes.c_void_p(shard.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                            int(shard.shape[0]), int(shard.shape[1]), int(iters), arr, int(rank),
                                            len(ptrs), fn, None, ctypes.c_void_p(stream.cuda_stream))
        if errors:
            raise errors[0]
        _check(status, "pe_polar_split_peers")
        return out

    def attach_comm(self, unique_id, rank, world):
        """pe_attach_comm: collective over `world` ranks (ncclCommInitRank)."""
        if len(unique_id) != 128:
            raise ValueError("unique_id must be the 128 bytes pe_nccl_unique_id returned")
        _check(lib().pe_attach_comm(self._h, ctypes.create_string_buffer(bytes(unique_id), 128), int(rank),
                                    int(world)), "pe_attach_comm")

    def attach_exchange(self, rank, world, fn):
        """pe_attach_exchange: pe_polar_sharded exchanges through the Python
        callable fn(op, ptr, nbytes, root, stream) (op PE_EXCHANGE_ALLGATHER /
        PE_EXCHANGE_BROADCAST, ptr an integer device address, stream a
        cudaStream_t handle) instead of NCCL; it raises on failure."""
        self._x_errors = []

        def cb(op, buf, nbytes, root, user, st):
            try:
                fn(int(op), int(buf or 0), int(nbytes), int(root), int(st or 0))
                return 0
            except Exception as e:          # reported when pe_polar_sharded returns
                self._x_errors.append(e)
                return 5                    # PE_ERR_NCCL
        self._xfn = EXCHANGE_FN(cb)         # kept alive as long as the context uses it
        _check(lib().pe_attach_exchange(self._h, int(rank), int(world), self._xfn, None), "pe_attach_exchange")

    def comm_info(self):
        r, w = ctypes.c_int(), ctypes.c_int()
        _check(lib().pe_comm_info(self._h, ctypes.byref(r), ctypes.byref(w)), "pe_comm_info")
        return r.value, w.value

    def polar_sharded(self, inputs, outputs, iters=5, stream=None):
        """pe_polar_sharded: every rank passes the whole layer set (same shapes
        on every rank); this rank computes its pe_shard_plan share and the
        results reach every rank's `outputs` (one all-gather per bucket when
        `outputs` are the views of dist.sharded_outputs, else per-matrix
        broadcasts).
        ``inputs[i]`` may be None on ranks that do not own matrix i."""
        import torch
        n = len(outputs)
        if len(inputs) != n:
            raise ValueError("polar_sharded takes equally long input / output lists")
        if n == 0:
            _check(lib().pe_polar_sharded(self._h, None, None, None, 0, int(iters), PE_BF16, None),
                   "pe_polar_sharded")
            return outputs
        dt = _dtype_code(outputs[0])
        for x, y in zip(inputs, outputs):
            if y.dim() != 2 or not y.is_contiguous() or not y.is_cuda or _dtype_code(y) != dt:
                raise ValueError("polar_sharded takes contiguous 2-D CUDA tensors of one dtype")
            if x is not None and (x.shape != y.shape or not x.is_contiguous() or _dtype_code(x) != dt):
                raise ValueError("polar_sharded: input / output shapes or dtypes differ")
        ins = (ctypes.c_void_p * n)(*[x.data_ptr() if x is not None else 0 for x in inputs])
        outs = (ctypes.c_void_p * n)(*[y.data_ptr() for y in outputs])
        shp = _shapes_arr([tuple(y.shape) for y in outputs])
        if stream is None:
            stream = torch.cuda.current_stream(outputs[0].device)
        status = lib().pe_polar_sharded(self._h, ins, outs, shp, n, int(iters), dt,
                                        ctypes.c_void_p(stream.cuda_stream))
        errs = getattr(self, "_x_errors", None)
        if errs:
            e = errs[0]
            errs.clear()
            raise e
        _check(status, "pe_polar_sharded")
        return outputs

    def sharded_exchange(self, outputs, stream=None):
        """pe_sharded_exchange: pe_polar_sharded's exchange step alone (the
        owned outputs already hold their results)."""
        import torch
        n = len(outputs)
        outs = (ctypes.c_void_p * max(n, 1))(*[y.data_ptr() for y in outputs])
        shp = _shapes_arr([tuple(y.shape) for y in outputs])
        if stream is None:
            stream = torch.cuda.current_stream(outputs[0].device)
        status = lib().pe_sharded_exchange(self._h, outs, shp, n, _dtype_code(outputs[0]),
                                           ctypes.c_void_p(stream.cuda_stream))
        errs = getattr(self, "_x_errors", None)
        if errs:
            e = errs[0]
            errs.clear()
            raise e
        _check(status, "pe_sharded_exchange")
        return outputs

    def polar_host(self, inputs, outputs, iters=5, stream=None):
        """pe_polar_host on host (pinned) CPU tensors; synchronous."""
        import torch
        n = len(inputs)
        if n == 0:
            return outputs
        dt = _dtype_code(inputs[0])
        ins = (ctypes.c_void_p * n)(*[x.data_ptr() for x in inputs])
        outs = (ctypes.c_void_p * n)(*[y.data_ptr() for y in outputs])
        shp = _shapes_arr([tuple(x.shape) for x in inputs])
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        _check(lib().pe_polar_host(self._h, ins, outs, shp, n, int(iters), dt,
                                   ctypes.c_void_p(stream.cuda_stream)), "pe_polar_host")
        return outputs


_default_ctx = {}


def _ctx_for(device):
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


def pe_polar(inputs, outputs=None, iters=5, coeffs=None, stream=None):
    """Module-level pe_polar on a per-device default context."""
    dev = inputs[0].device.index if inputs else 0
    ctx = _ctx_for(dev or 0)
    if coeffs is not None:
        ctx.set_coeffs(coeffs)
    return ctx.polar(inputs, outputs, iters, stream)


def pe_polar_host(inputs, outputs, iters=5, device=0, stream=None):
    return _ctx_for(device).polar_host(inputs, outputs, iters, stream)


class MuonPE:
    """Muon with Polar Express as the polar step: a minimal
    optimizer over bf16 2-D CUDA parameters whose whole step -- momentum
    M <- beta M + (1 - beta) G, X = polar(M) by Polar Express, W <- W - lr X --
    is one pe_muon_step call (momentum fused into the norm pass, the weight
    update into the last update epilogue).  Parameters of other shapes or
    dtypes are the caller's business (the paper optimises them with AdamW,
    P:393).  Usage: opt = MuonPE(params, lr=0.02, beta=0.9); loss.backward();
    opt.step()."""

    def __init__(self, params, lr=0.02, beta=0.9, iters=5, device=None):
        import torch
        self.params = [p for p in params]
        for p in self.params:
            if p.dim() != 2 or p.dtype != torch.bfloat16 or not p.is_cuda or not p.is_contiguous():
                raise ValueError("MuonPE takes contiguous 2-D bf16 CUDA parameters")
        self.lr, self.beta, self.iters = float(lr), float(beta), int(iters)
        self.momenta = [torch.zeros_like(p) for p in self.params]     # M_0 = 0
        dev = self.params[0].device.index if self.params else (device or 0)
        self.ctx = Context(dev or 0)
        if self.params:
            self.ctx.reserve([tuple(p.shape) for p in self.params])

    def step(self):
        import torch
        live = [(p, m) for p, m in zip(self.params, self.momenta) if p.grad is not None]
        if not live:
            return
        with torch.no_grad():
            grads = [p.grad.to(torch.bfloat16).contiguous() for p, _ in live]
            self.ctx.muon_step([p.data for p, _ in live], [m for _, m in live], grads, beta=self.beta, lr=self.lr,
                               iters=self.iters)

    def zero_grad(self, set_to_none=True):
        for p in self.params:
            if set_to_none:
                p.grad = None
            elif p.grad is not None:
                p.grad.zero_()
