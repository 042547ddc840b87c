"""Thin ctypes binding of libnmt.so (include/nmt.h).  Argument marshalling only: every step of the
hot path runs in the library's CUDA kernels.  There is no fallback: if libnmt.so is missing or
no sm_100 GPU is present the calls raise."""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NMT_LIB_PATH") or os.path.join(_HERE, "libnmt.so")  # (override: A/B builds)

NMT_PREC_FP32CLASS = 0
NMT_PREC_BF16 = 1
PRECISIONS = {"fp32class": NMT_PREC_FP32CLASS, "bf16": NMT_PREC_BF16}

STATUS = {0: "NMT_OK", 1: "NMT_ERR_INVALID_ARG", 2: "NMT_ERR_IO", 3: "NMT_ERR_FORMAT", 4: "NMT_ERR_MISSING_PARAM",
          5: "NMT_ERR_SHAPE", 6: "NMT_ERR_EMPTY_SOURCE", 7: "NMT_ERR_TOKEN_RANGE", 8: "NMT_ERR_BAD_STATE",
          9: "NMT_ERR_CAPACITY", 10: "NMT_ERR_CUDA", 11: "NMT_ERR_NCCL", 12: "NMT_ERR_OOM"}

# every symbol include/nmt.h declares (checked by tests/test_abi.py)
EXPORTS = ["nmt_last_error", "nmt_load", "nmt_load_buffer", "nmt_model_dims", "nmt_model_free", "nmt_encode",
           "nmt_root", "nmt_ctx_free", "nmt_score_batch", "nmt_score_forest", "nmt_score_batch_dev", "nmt_ctx_check", "nmt_ctx_stats",
           "nmt_inject_states", "nmt_logprobs_full", "nmt_debug_encoder", "nmt_debug_intermediates",
           "nmt_test_gemm", "nmt_encode_dev", "nmt_inject_states_dev", "nmt_launch_count", "nmt_profile",
           "nmt_profile_read", "nmt_bench_gemm", "nmt_ensemble_init", "nmt_ensemble_get_unique_id", "nmt_ensemble_combine",
           "nmt_ensemble_free", "nmt_params_average", "nmt_beam_step",
           "nmt_encode_batch", "nmt_save_params", "nmt_params_bytes", "nmt_random_params", "nmt_create_random",
           "nmt_debug_vocab", "nmt_score_batch_multi", "nmt_ctx_reserve", "nmt_score_sequences",
           "nmt_vocab_shard", "nmt_debug_vocab_shards", "nmt_score_forest_multi", "nmt_ensemble_init_local",
           "nmt_model_memory", "nmt_device_allocations", "nmt_debug_live_objects"]


N_STAGES = 19
STAGES = ["plan", "gather", "gemm_h1", "gru1", "gemm_q", "attention", "gemm_g2", "gru2", "gemm_ro", "readout",
          "vocab_gemm_lse", "finalize", "gather_dot", "enc_gather", "enc_gemm_in", "enc_recurrence", "enc_init",
          "enc_pctx", "inject"]


def device_allocations() -> Tuple[int, int]:
    """nmt_device_allocations: (count, bytes) of the library's live device allocations."""
    n, b = C.c_int64(), C.c_size_t()
    _check(lib().nmt_device_allocations(C.byref(n), C.byref(b)))
    return n.value, b.value


def live_objects() -> Tuple[int, int]:
    """nmt_debug_live_objects: (models, contexts incl. pooled) that exist in the process."""
    a, b = C.c_int64(), C.c_int64()
    _check(lib().nmt_debug_live_objects(C.byref(a), C.byref(b)))
    return a.value, b.value


def launch_count() -> int:
    return int(lib().nmt_launch_count())


def params_average(blobs, device: int = 0) -> bytes:
    """nmt_params_average: element-wise average of n params containers (NMT-k-Avg)."""
    blobs = [bytes(b) for b in blobs]
    n = len(blobs)
    bufs = (C.c_char_p * n)(*blobs)
    lens = (C.c_size_t * n)(*[len(b) for b in blobs])
    out = C.create_string_buffer(len(blobs[0]) if n else 0)
    _check(lib().nmt_params_average(n, C.cast(bufs, C.c_void_p), C.cast(lens, C.c_void_p), device, out,
                                    len(blobs[0]) if n else 0))
    return out.raw


READOUTS = {"tanh": 0, "maxout": 1}


def random_params(dim_emb: int, dim_hid: int, vocab_src: int, vocab_tgt: int, readout: str = "tanh",
                  seed: int = 0, logit_std: float = 1.0) -> bytes:
    """nmt_random_params: the seeded synthetic params container (host only, no GPU needed)."""
    d = Dims(dim_emb, dim_hid, vocab_src, vocab_tgt, 0, READOUTS[readout])
    n = C.c_size_t(0)
    _check(lib().nmt_random_params(C.byref(d), seed, logit_std, None, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    _check(lib().nmt_random_params(C.byref(d), seed, logit_std, C.cast(buf, C.c_void_p), C.byref(n)))
    return buf.raw[:n.value]


def score_batch_multi(contexts, parents, cand_offsets, cand_words, with_argmax: bool = True):
    """nmt_score_batch_multi: parent k belongs to contexts[k] (all of one model)."""
    n = len(parents)
    if isinstance(contexts, np.ndarray):  # int64 handles (Context.handle), e.g. built with np.repeat
        hs = np.ascontiguousarray(contexts, dtype=np.int64)
        hs_ptr = _ptr(hs)
    else:
        hs = (C.c_void_p * max(n, 1))(*[c._h.value for c in contexts])
        hs_ptr = C.cast(hs, C.c_void_p)
    par = _c(parents, np.int64)
    off = _c(cand_offsets, np.int32)
    words = _c(cand_words, np.int32)
    nc = int(off[-1]) if len(off) else 0
    logp = np.empty(nc, np.float32)
    child = np.empty(nc, np.int64)
    am = np.empty(n, np.int32) if with_argmax else None
    _check(lib().nmt_score_batch_multi(n, hs_ptr, _ptr(par), _ptr(off), _ptr(words), _ptr(logp),
                                       _ptr(child), _ptr(am)))
    return logp, child, am


def score_forest_multi(contexts, hyp_states, phrase_offsets, phrase_words):
    """nmt_score_forest_multi: pair i expands hyp_states[i] of contexts[i] (Context objects or int64
    handles) by its phrase; returns (summed log-probs [n], final states [n])."""
    n = len(hyp_states)
    if isinstance(contexts, np.ndarray):
        hs = np.ascontiguousarray(contexts, dtype=np.int64)
    else:
        hs = np.array([c._h.value for c in contexts], np.int64)
    st = _c(hyp_states, np.int64)
    off = _c(phrase_offsets, np.int32)
    w = _c(phrase_words, np.int32)
    lp = np.empty(n, np.float32)
    out = np.empty(n, np.int64)
    _check(lib().nmt_score_forest_multi(n, _ptr(hs), _ptr(st), _ptr(off), _ptr(w), _ptr(lp), _ptr(out)))
    return lp, out


class NmtError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class Dims(C.Structure):
    _fields_ = [("dim_emb", C.c_int32), ("dim_hid", C.c_int32), ("vocab_src", C.c_int32), ("vocab_tgt", C.c_int32),
                ("max_src_len", C.c_int32), ("readout", C.c_int32)]


DEV_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p, C.c_void_p)
DEV_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p, C.c_void_p)


class Opts(C.Structure):
    _fields_ = [("device", C.c_int32), ("precision", C.c_int32), ("max_src_len", C.c_int32), ("stream", C.c_void_p),
                ("arena_bytes", C.c_size_t), ("dev_alloc", DEV_ALLOC_FN), ("dev_free", DEV_FREE_FN),
                ("alloc_ctx", C.c_void_p)]


# PyTorch's caching allocator as the library's device allocator (include/nmt.h nmt_opts.dev_alloc):
# the library's weights, workspaces and state arenas then show up in torch.cuda.memory_allocated()
# and share torch's cache.  Called back from inside nmt_* calls (ctypes re-acquires the GIL).
def _torch_alloc(nbytes, device, stream, ctx):
    try:
        import torch
        return int(torch.cuda.caching_allocator_alloc(int(nbytes), int(device), int(stream or 0)))
    except Exception:  # noqa: BLE001  (out of memory -> NULL -> NMT_ERR_OOM)
        return None


def _torch_free(ptr, nbytes, device, stream, ctx):
    try:
        import torch
        torch.cuda.caching_allocator_delete(int(ptr))
    except Exception:  # noqa: BLE001
        pass


_TORCH_ALLOC = DEV_ALLOC_FN(_torch_alloc)
_TORCH_FREE = DEV_FREE_FN(_torch_free)

# models and contexts alive in this process: released before interpreter teardown (the torch
# allocator callbacks must not run after torch has gone)
import atexit  # noqa: E402
import weakref  # noqa: E402

_LIVE = weakref.WeakSet()


@atexit.register
def _close_all():
    for o in sorted(list(_LIVE), key=lambda x: 0 if isinstance(x, Context) else 1):
        try:
            o.close()
        except Exception:  # noqa: BLE001
            pass


def _make_opts(device, precision, max_src_len, stream, allocator, arena_bytes) -> Opts:
    if allocator == "auto":
        import sys
        allocator = "torch" if "torch" in sys.modules else None
    if allocator == "torch":
        return Opts(device, PRECISIONS[precision], max_src_len, stream, arena_bytes, _TORCH_ALLOC, _TORCH_FREE, None)
    if allocator is not None:
        raise ValueError("allocator must be 'torch', 'auto' or None")
    return Opts(device, PRECISIONS[precision], max_src_len, stream, arena_bytes, DEV_ALLOC_FN(), DEV_FREE_FN(), None)


_lib = None


def _torch_nccl_path() -> Optional[str]:
    """Path of the NCCL that torch links (pip package nvidia-nccl), found without importing torch."""
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return None
    for d in (spec.submodule_search_locations or []) if spec else []:
        p = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(p):
            return p
    return None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built (run python -m paper_1605_04809_b200.build)")
        if "NMT_NCCL_LIB" not in os.environ:  # ensemble hook: the same NCCL as torch (ensemble.cu)
            p = _torch_nccl_path()
            if p:
                os.environ["NMT_NCCL_LIB"] = p
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, f32p = C.c_void_p, C.c_int32, C.c_int64, C.c_void_p
        sig = {
            "nmt_last_error": (C.c_char_p, []),
            "nmt_load": (i32, [C.c_char_p, C.POINTER(Opts), C.POINTER(vp)]),
            "nmt_load_buffer": (i32, [vp, C.c_size_t, C.POINTER(Opts), C.POINTER(vp)]),
            "nmt_model_dims": (i32, [vp, C.POINTER(Dims)]),
            "nmt_device_allocations": (i32, [C.POINTER(C.c_int64), C.POINTER(C.c_size_t)]),
            "nmt_debug_live_objects": (i32, [C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
            "nmt_model_memory": (i32, [vp, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
            "nmt_model_free": (None, [vp]),
            "nmt_encode": (i32, [vp, vp, i32, C.POINTER(vp)]),
            "nmt_root": (i64, [vp]),
            "nmt_ctx_free": (None, [vp]),
            "nmt_score_batch": (i32, [vp, i32, vp, vp, vp, vp, vp, vp]),
            "nmt_score_batch_dev": (i32, [vp, i32, vp, vp, i32, vp, vp, vp, vp]),
            "nmt_score_forest": (i32, [vp, i32, vp, vp, vp, vp, vp, vp]),
            "nmt_ctx_check": (i32, [vp]),
            "nmt_ctx_stats": (i32, [vp, C.POINTER(i64), C.POINTER(i64)]),
            "nmt_inject_states": (i32, [vp, i32, vp, vp, vp]),
            "nmt_logprobs_full": (i32, [vp, i64, vp]),
            "nmt_debug_encoder": (i32, [vp, vp, vp, vp]),
            "nmt_debug_intermediates": (i32, [vp, i64, vp, vp, vp, vp, vp, vp, vp]),
            "nmt_test_gemm": (i32, [i32, i32, i32, i32, vp, vp, vp, vp]),
            "nmt_ensemble_init": (i32, [i32, i32, vp, i32, C.POINTER(vp)]),
            "nmt_ensemble_get_unique_id": (i32, [vp]),
            "nmt_ensemble_init_local": (i32, [i32, vp, vp]),
            "nmt_ensemble_combine": (i32, [vp, vp, i32, C.c_float, i32, i32, vp, vp]),
            "nmt_ensemble_free": (None, [vp]),
            "nmt_encode_dev": (i32, [vp, vp, i32, C.POINTER(vp)]),
            "nmt_inject_states_dev": (i32, [vp, i32, vp, vp, vp]),
            "nmt_launch_count": (C.c_longlong, []),
            "nmt_profile": (i32, [vp, i32]),
            "nmt_profile_read": (i32, [vp, vp, vp]),
            "nmt_bench_gemm": (i32, [i32, i32, i32, i32, i32, i32, i32, C.POINTER(C.c_float)]),
            "nmt_params_average": (i32, [i32, vp, vp, i32, vp, C.c_size_t]),
            "nmt_beam_step": (i32, [vp, i32, vp, i32, vp, vp, vp]),
            "nmt_encode_batch": (i32, [vp, i32, vp, vp, vp]),
            "nmt_save_params": (i32, [vp, C.c_char_p]),
            "nmt_params_bytes": (i32, [vp, vp, C.POINTER(C.c_size_t)]),
            "nmt_random_params": (i32, [C.POINTER(Dims), C.c_uint64, C.c_float, vp, C.POINTER(C.c_size_t)]),
            "nmt_create_random": (i32, [C.POINTER(Dims), C.c_uint64, C.c_float, C.POINTER(Opts), C.POINTER(vp)]),
            "nmt_debug_vocab": (i32, [vp, i32, vp, vp, vp, vp, vp, vp]),
            "nmt_score_batch_multi": (i32, [i32, vp, vp, vp, vp, vp, vp, vp]),
            "nmt_ctx_reserve": (i32, [vp, i64, i64]),
            "nmt_score_sequences": (i32, [vp, i32, vp, vp, vp, vp]),
            "nmt_vocab_shard": (i32, [vp, i32, i32, vp]),
            "nmt_score_forest_multi": (i32, [i32, vp, vp, vp, vp, vp, vp]),
            "nmt_debug_vocab_shards": (i32, [vp, i32, vp, i32, vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status != 0:
        raise NmtError(status, lib().nmt_last_error().decode(errors="replace"))


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=dtype)


class Model:
    """nmt_load / nmt_load_buffer.  `params` is a path or the bytes of a params container."""

    def __init__(self, params, precision: str = "bf16", device: int = 0, max_src_len: int = 64,
                 stream: Optional[int] = None, allocator: Optional[str] = "auto", arena_bytes: int = 0):
        """allocator: "torch" (PyTorch's caching allocator), None (the library's private pool) or
        "auto" (torch when it is imported).  arena_bytes: state-arena budget (0 = unbounded)."""
        self._h = C.c_void_p()
        opts = _make_opts(device, precision, max_src_len, stream, allocator, arena_bytes)
        if isinstance(params, (bytes, bytearray, memoryview)):
            buf = (C.c_char * len(params)).from_buffer_copy(params)
            _check(lib().nmt_load_buffer(C.cast(buf, C.c_void_p), len(params), C.byref(opts), C.byref(self._h)))
        else:
            _check(lib().nmt_load(str(params).encode(), C.byref(opts), C.byref(self._h)))
        d = Dims()
        _check(lib().nmt_model_dims(self._h, C.byref(d)))
        self.dims = d
        self.precision = precision
        _LIVE.add(self)

    def memory(self) -> dict:
        """nmt_model_memory: device bytes held now / at peak, and state-arena bytes."""
        a, b, c = C.c_size_t(), C.c_size_t(), C.c_size_t()
        _check(lib().nmt_model_memory(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return {"live": a.value, "peak": b.value, "arena": c.value}

    def encode(self, src_ids: Sequence[int]) -> "Context":
        return Context(self, src_ids)

    @classmethod
    def create_random(cls, dim_emb: int, dim_hid: int, vocab_src: int, vocab_tgt: int, readout: str = "tanh",
                      seed: int = 0, logit_std: float = 1.0, precision: str = "bf16", device: int = 0,
                      max_src_len: int = 64, allocator: Optional[str] = "auto") -> "Model":
        """nmt_create_random: the seeded synthetic model generated and loaded by the library."""
        m = cls.__new__(cls)
        m._h = C.c_void_p()
        d = Dims(dim_emb, dim_hid, vocab_src, vocab_tgt, max_src_len, READOUTS[readout])
        opts = _make_opts(device, precision, max_src_len, None, allocator, 0)
        _check(lib().nmt_create_random(C.byref(d), seed, logit_std, C.byref(opts), C.byref(m._h)))
        dd = Dims()
        _check(lib().nmt_model_dims(m._h, C.byref(dd)))
        m.dims = dd
        m.precision = precision
        _LIVE.add(m)
        return m

    def save_params(self, path: str) -> None:
        _check(lib().nmt_save_params(self._h, str(path).encode()))

    def params_bytes(self) -> bytes:
        n = C.c_size_t(0)
        _check(lib().nmt_params_bytes(self._h, None, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _check(lib().nmt_params_bytes(self._h, C.cast(buf, C.c_void_p), C.byref(n)))
        return buf.raw[:n.value]

    def debug_vocab(self, t: np.ndarray, cand_offsets, cand_words):
        """nmt_debug_vocab: the vocabulary stage alone on given readout outputs t [R x E]."""
        t = _c(t, np.float32)
        R = t.shape[0]
        off = _c(cand_offsets, np.int32)
        words = _c(cand_words, np.int32)
        nc = int(off[-1]) if len(off) else 0
        logp = np.empty(nc, np.float32)
        logZ = np.empty(R, np.float32)
        am = np.empty(R, np.int32)
        _check(lib().nmt_debug_vocab(self._h, R, _ptr(t), _ptr(off), _ptr(words), _ptr(logp), _ptr(logZ), _ptr(am)))
        return logp, logZ, am

    def vocab_shard(self, rank: int, world: int, comm: Optional["Ensemble"]) -> None:
        """nmt_vocab_shard: vocab-parallel scoring over `world` ranks (comm = an Ensemble communicator)."""
        _check(lib().nmt_vocab_shard(self._h, rank, world, comm._h if comm is not None else None))

    def debug_vocab_shards(self, t: np.ndarray, n_slices: int):
        """nmt_debug_vocab_shards: the vocab-parallel combine emulated with n_slices slices."""
        t = _c(t, np.float32)
        R = t.shape[0]
        logZ = np.empty(R, np.float32)
        am = np.empty(R, np.int32)
        _check(lib().nmt_debug_vocab_shards(self._h, R, _ptr(t), n_slices, _ptr(logZ), _ptr(am)))
        return logZ, am

    def encode_batch(self, sources: Sequence[Sequence[int]]) -> list:
        """nmt_encode_batch: one context per source, all recurrences advanced together."""
        srcs = [_c(x, np.int32) for x in sources]
        n = len(srcs)
        if n == 0:
            return []
        ids = np.concatenate(srcs).astype(np.int32) if sum(len(x) for x in srcs) else np.zeros(1, np.int32)
        off = np.zeros(n + 1, np.int32)
        off[1:] = np.cumsum([len(x) for x in srcs])
        hs = (C.c_void_p * n)()
        _check(lib().nmt_encode_batch(self._h, n, _ptr(ids), _ptr(off), C.cast(hs, C.c_void_p)))
        return [Context._wrap(self, hs[i], len(srcs[i])) for i in range(n)]

    def encode_dev(self, src_ptr: int, length: int) -> "Context":
        """nmt_encode_dev: source ids already resident in device memory (int32)."""
        return Context(self, None, dev=(src_ptr, length))

    def profile(self, mode: int) -> None:
        _check(lib().nmt_profile(self._h, mode))

    def profile_read(self) -> Tuple[np.ndarray, np.ndarray]:
        ms = np.zeros(N_STAGES, np.float64)
        cnt = np.zeros(N_STAGES, np.int64)
        _check(lib().nmt_profile_read(self._h, _ptr(ms), _ptr(cnt)))
        return ms, cnt

    def close(self):
        if self._h:
            lib().nmt_model_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """nmt_encode: the source context and its state arena (root node = (s0, BOS))."""

    def __init__(self, model: Model, src_ids: Optional[Sequence[int]], dev: Optional[Tuple[int, int]] = None):
        self.model = model
        self._h = C.c_void_p()
        if dev is not None:
            _check(lib().nmt_encode_dev(model._h, dev[0], dev[1], C.byref(self._h)))
            self.Tx = dev[1]
        else:
            src = _c(src_ids, np.int32)
            _check(lib().nmt_encode(model._h, _ptr(src), len(src), C.byref(self._h)))
            self.Tx = len(src)
        self.root = int(lib().nmt_root(self._h))
        _LIVE.add(self)

    @property
    def handle(self) -> int:
        return int(self._h.value)

    @classmethod
    def _wrap(cls, model: Model, handle: int, Tx: int) -> "Context":
        c = cls.__new__(cls)
        c.model = model
        c._h = C.c_void_p(handle)
        c.Tx = Tx
        c.root = int(lib().nmt_root(c._h))
        _LIVE.add(c)
        return c

    def score_batch(self, parents, cand_offsets, cand_words, with_argmax: bool = True
                    ) -> Tuple[np.ndarray, np.ndarray, Optional[np.ndarray]]:
        par = _c(parents, np.int64)
        off = _c(cand_offsets, np.int32)
        words = _c(cand_words, np.int32)
        n = int(off[-1]) if len(off) else 0
        logp = np.empty(n, np.float32)
        child = np.empty(n, np.int64)
        am = np.empty(len(par), np.int32) if with_argmax else None
        _check(lib().nmt_score_batch(self._h, len(par), _ptr(par), _ptr(off), _ptr(words), _ptr(logp), _ptr(child),
                                     _ptr(am)))
        return logp, child, am

    def beam_step(self, parents, k: int) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        """nmt_beam_step: the k best next words of each parent over the whole vocabulary
        -> (words [n, k], logprob [n, k], child [n, k]), descending log-prob per parent."""
        par = _c(parents, np.int64)
        n = len(par)
        words = np.empty((n, k), np.int32)
        logp = np.empty((n, k), np.float32)
        child = np.empty((n, k), np.int64)
        _check(lib().nmt_beam_step(self._h, n, _ptr(par), k, _ptr(words), _ptr(logp), _ptr(child)))
        return words, logp, child

    def score_batch_dev(self, n_parents: int, parents_ptr: int, offsets_ptr: int, n_cand: int, words_ptr: int,
                        logp_ptr: int, child_ptr: int, argmax_ptr: Optional[int] = None) -> None:
        """Device-resident variant (int32 device arrays, e.g. torch tensors' data_ptr())."""
        _check(lib().nmt_score_batch_dev(self._h, n_parents, parents_ptr, offsets_ptr, n_cand, words_ptr, logp_ptr,
                                         child_ptr, argmax_ptr))

    def score_forest(self, hyp_states, phrase_offsets, phrase_words):
        """nmt_score_forest: ScoreBatch over (hypothesis, phrase) pairs in one call.
        Returns (summed log-probs [n], final states [n], stats dict)."""
        hs = _c(hyp_states, np.int64)
        off = _c(phrase_offsets, np.int32)
        w = _c(phrase_words, np.int32)
        n = len(hs)
        lp = np.empty(n, np.float32)
        st = np.empty(n, np.int64)
        stats = np.zeros(33, np.int32)
        _check(lib().nmt_score_forest(self._h, n, _ptr(hs), _ptr(off), _ptr(w), _ptr(lp), _ptr(st), _ptr(stats)))
        steps = int(stats[0])
        return lp, st, {"steps": steps, "edges_per_depth": stats[1:1 + steps].tolist(),
                        "rows_per_depth": stats[17:17 + steps].tolist()}

    def score_sequences(self, sequences) -> Tuple[np.ndarray, np.ndarray]:
        """nmt_score_sequences: n-best forced rescoring from the root; (sum log-prob, final state)."""
        seqs = [_c(x, np.int32) for x in sequences]
        n = len(seqs)
        off = np.zeros(n + 1, np.int32)
        off[1:] = np.cumsum([len(x) for x in seqs])
        w = np.concatenate(seqs).astype(np.int32) if n else np.zeros(1, np.int32)
        lp = np.empty(n, np.float32)
        st = np.empty(n, np.int64)
        _check(lib().nmt_score_sequences(self._h, n, _ptr(off), _ptr(w), _ptr(lp), _ptr(st)))
        return lp, st

    def check(self) -> None:
        _check(lib().nmt_ctx_check(self._h))

    def reserve(self, n_nodes: int, n_stepped: int) -> None:
        _check(lib().nmt_ctx_reserve(self._h, n_nodes, n_stepped))

    def stats(self) -> Tuple[int, int]:
        a, b = C.c_int64(), C.c_int64()
        _check(lib().nmt_ctx_stats(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def inject_states(self, s: np.ndarray, y_prev: Sequence[int]) -> np.ndarray:
        s = _c(s, np.float32)
        y = _c(y_prev, np.int32)
        out = np.empty(len(y), np.int64)
        _check(lib().nmt_inject_states(self._h, len(y), _ptr(s), _ptr(y), _ptr(out)))
        return out

    def inject_states_dev(self, n: int, s_ptr: int, y_ptr: int, out_ptr: int) -> None:
        _check(lib().nmt_inject_states_dev(self._h, n, s_ptr, y_ptr, out_ptr))

    def logprobs_full(self, node: int) -> np.ndarray:
        out = np.empty(self.model.dims.vocab_tgt, np.float32)
        _check(lib().nmt_logprobs_full(self._h, int(node), _ptr(out)))
        return out

    def debug_encoder(self):
        H = self.model.dims.dim_hid
        ctx = np.empty((self.Tx, 2 * H), np.float32)
        pctx = np.empty((self.Tx, 2 * H), np.float32)
        s0 = np.empty(H, np.float32)
        _check(lib().nmt_debug_encoder(self._h, _ptr(ctx), _ptr(pctx), _ptr(s0)))
        return ctx, pctx, s0

    def debug_intermediates(self, node: int) -> dict:
        d = self.model.dims
        H, E = d.dim_hid, d.dim_emb
        out = dict(s1=np.empty(H, np.float32), alpha=np.empty(self.Tx, np.float32), c=np.empty(2 * H, np.float32),
                   s2=np.empty(H, np.float32), t=np.empty(E, np.float32), logZ=np.empty(1, np.float32),
                   argmax=np.empty(1, np.int32))
        _check(lib().nmt_debug_intermediates(self._h, int(node), *[_ptr(out[k]) for k in
                                                                    ("s1", "alpha", "c", "s2", "t", "logZ", "argmax")]))
        return out

    def close(self):
        if self._h:
            lib().nmt_ctx_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def test_gemm(A: np.ndarray, B: np.ndarray, bias: Optional[np.ndarray] = None, split: bool = False) -> np.ndarray:
    A = _c(A, np.float32)
    B = _c(B, np.float32)
    M, K = A.shape
    N = B.shape[1]
    out = np.empty((M, N), np.float32)
    b = None if bias is None else _c(bias, np.float32)
    _check(lib().nmt_test_gemm(M, N, K, int(split), _ptr(A), _ptr(B), _ptr(b), _ptr(out)))
    return out


def bench_gemm(M: int, N: int, K: int, split: bool = False, epi: int = 0, ksplit: int = 1, iters: int = 20) -> float:
    """Average milliseconds of the tcgen05 GEMM engine on device-resident operands (tuning aid)."""
    ms = C.c_float()
    _check(lib().nmt_bench_gemm(M, N, K, int(split), epi, ksplit, iters, C.byref(ms)))
    return ms.value


class Ensemble:
    """nmt_ensemble_*: one member per GPU/process; NCCL reduce of per-word scores to the root."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_char * 128)()
        _check(lib().nmt_ensemble_get_unique_id(C.cast(buf, C.c_void_p)))
        return bytes(buf)

    def __init__(self, n_members: int, rank: int, unique_id: bytes, device: int):
        self._h = C.c_void_p()
        self.n_members, self.rank = n_members, rank
        buf = (C.c_char * 128).from_buffer_copy(unique_id)
        _check(lib().nmt_ensemble_init(n_members, rank, C.cast(buf, C.c_void_p), device, C.byref(self._h)))

    @classmethod
    def local(cls, n_members: int, devices: Optional[Sequence[int]] = None) -> list:
        """nmt_ensemble_init_local: n communicator handles of one in-process group (rank q = item q);
        drive each member from its own thread."""
        hs = (C.c_void_p * n_members)()
        devs = None if devices is None else _c(devices, np.int32)
        _check(lib().nmt_ensemble_init_local(n_members, _ptr(devs), C.cast(hs, C.c_void_p)))
        out = []
        for q in range(n_members):
            e = cls.__new__(cls)
            e._h = C.c_void_p(hs[q])
            e.n_members, e.rank = n_members, q
            out.append(e)
        return out

    def combine(self, logp_ptr: int, n: int, weight: float, mode: int, root: int, out_ptr: Optional[int],
                stream: Optional[int] = None) -> None:
        _check(lib().nmt_ensemble_combine(self._h, logp_ptr, n, weight, mode, root, out_ptr, stream))

    def close(self):
        if self._h:
            lib().nmt_ensemble_free(self._h)
            self._h = C.c_void_p()
