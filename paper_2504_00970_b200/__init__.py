"""SentenceKV hot path on B200 (sm_100a) -- thin Python binding of ``libsentencekv.so``.

The C ABI is declared in ``include/sentencekv.h``; this module only marshals arguments
(torch tensors -> device pointers, torch streams -> cudaStream_t) and raises on a non-OK
status.  Every step of the path (P1 segmentation, P2 Eq. 1 embeddings, D1 scoring, D2 budgeted
selection, D3 gather, D4 Eq. 3 attention) runs in the library's CUDA kernels.  There is no CPU
fallback: importing this package fails if the library is missing or cannot be loaded.

Functions keep the ABI names (``sentencekv_create``, ``sentencekv_prefill_compress``,
``sentencekv_decode_select``, ``sentencekv_decode_attend``, ...); ``SentenceKV`` bundles them
around one context.
"""
from __future__ import annotations

import ctypes
import os

import torch

__all__ = [
    "SkvConfig", "SkvError", "SentenceKV", "lib", "LIB_PATH",
    "SKV_KV_DEVICE", "SKV_KV_HOST", "sentencekv_config_default", "sentencekv_create", "sentencekv_destroy",
    "sentencekv_prefill_compress", "sentencekv_decode_select", "sentencekv_decode_attend", "sentencekv_decode_step",
    "sentencekv_sync",
]

LIB_PATH = os.environ.get("SKV_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsentencekv.so")

SKV_OK, SKV_ERR_INVALID_ARGUMENT, SKV_ERR_STATE, SKV_ERR_UNSUPPORTED, SKV_ERR_CUDA, SKV_ERR_OUT_OF_MEMORY = range(6)
SKV_KV_DEVICE, SKV_KV_HOST = 0, 1
SKV_BUCKETS_SENTENCE, SKV_BUCKETS_EQUAL, SKV_BUCKETS_QUEST = 0, 1, 2
SKV_QUERY_MEAN, SKV_QUERY_CURRENT = 0, 1
SKV_FILL_PREFIX, SKV_FILL_SKIP = 0, 1
_STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "STATE", 3: "UNSUPPORTED", 4: "CUDA", 5: "OUT_OF_MEMORY"}


class SkvConfig(ctypes.Structure):
    """Mirror of ``skv_config`` (include/sentencekv.h)."""

    _fields_ = [
        ("batch", ctypes.c_int32), ("layers", ctypes.c_int32), ("q_heads", ctypes.c_int32),
        ("kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("max_context", ctypes.c_int32),
        ("token_budget", ctypes.c_int32), ("semantic_factor", ctypes.c_float), ("obs_window", ctypes.c_int32),
        ("residency", ctypes.c_int32), ("device", ctypes.c_int32), ("kv_head_begin", ctypes.c_int32),
        ("kv_head_count", ctypes.c_int32), ("batch_begin", ctypes.c_int32), ("batch_count", ctypes.c_int32),
        ("bucket_mode", ctypes.c_int32), ("chunk_size", ctypes.c_int32), ("outlier_n", ctypes.c_float),
        ("query_mode", ctypes.c_int32), ("fill_mode", ctypes.c_int32), ("max_generated", ctypes.c_int32),
    ]


class SkvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"SKV_{_STATUS.get(status, status)}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a).  There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
    sig = {
        "sentencekv_config_default": (None, [ctypes.POINTER(SkvConfig)]),
        "sentencekv_create": (i32, [ctypes.POINTER(SkvConfig), ctypes.POINTER(P)]),
        "sentencekv_destroy": (i32, [P]),
        "sentencekv_last_error": (ctypes.c_char_p, [P]),
        "sentencekv_sync": (i32, [P]),
        "sentencekv_prefill_compress": (i32, [P, i32, P, i32, P, i32, P, P, f32, i32, P, P]),
        "sentencekv_decode_select": (i32, [P, i32, P, P, P, P, P, P]),
        "sentencekv_decode_attend": (i32, [P, i32, P, P, P]),
        "sentencekv_decode_step": (i32, [P, i32, P, P, P, P, P, P, P]),
        "sentencekv_decode_append": (i32, [P, i32, P, P, P, P]),
        "sentencekv_set_output_peers": (i32, [P, i32, i32, i32, P, P]),
        "sentencekv_wait_outputs": (i32, [P, i32, P]),
        "sentencekv_sentence_counts": (i32, [P, P]),
        "sentencekv_sentence_capacity": (i32, [P]),
        "sentencekv_copy_offsets": (i32, [P, P, P]),
        "sentencekv_copy_embeddings": (i32, [P, i32, P, P]),
        "sentencekv_copy_scores": (i32, [P, i32, P, P]),
        "sentencekv_launch_count": (i64, [P]),
        "sentencekv_set_profiling": (i32, [P, i32]),
        "sentencekv_set_band_log2": (i32, [P, i32]),
        "sentencekv_host_fetch_bytes": (i32, [P, i32, P]),
        "sentencekv_profile_read": (i32, [P, P, P]),
        "sentencekv_retained_tokens": (i32, [P, i32]),
        "sentencekv_copy_importance": (i32, [P, i32, P, P]),
        "sentencekv_copy_retained": (i32, [P, i32, P, P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    return L


lib = _load()


def _check(ctx, status: int):
    if status != SKV_OK:
        msg = lib.sentencekv_last_error(ctx).decode() if ctx else ""
        raise SkvError(status, msg)


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise ValueError("tensors passed to libsentencekv must be contiguous")
        return ctypes.c_void_p(t.data_ptr())
    return ctypes.c_void_p(int(t))


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


# ------------------------------------------------------------------ ABI-named functions


def sentencekv_config_default(**kw) -> SkvConfig:
    cfg = SkvConfig()
    lib.sentencekv_config_default(ctypes.byref(cfg))
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


def sentencekv_create(cfg: SkvConfig) -> ctypes.c_void_p:
    ctx = ctypes.c_void_p()
    st = lib.sentencekv_create(ctypes.byref(cfg), ctypes.byref(ctx))
    if st != SKV_OK:
        raise SkvError(st, "sentencekv_create rejected the configuration")
    return ctx


def sentencekv_destroy(ctx) -> None:
    _check(None, lib.sentencekv_destroy(ctx))


def sentencekv_sync(ctx) -> None:
    _check(ctx, lib.sentencekv_sync(ctx))


def sentencekv_prefill_compress(ctx, layer, token_ids, L, boundary_ids, K, V, semantic_factor, token_budget,
                                q_window=None, stream=None) -> None:
    """P1 (layer 0) + P2 (+ P3 in host residency); see include/sentencekv.h."""
    if boundary_ids is not None:
        ids = (ctypes.c_int32 * len(boundary_ids))(*[int(x) for x in boundary_ids])
        nb = len(boundary_ids)
    else:
        ids, nb = None, 0
    _check(ctx, lib.sentencekv_prefill_compress(ctx, int(layer), _ptr(token_ids), int(L), ids, nb, _ptr(K), _ptr(V),
                                                float(semantic_factor), int(token_budget), _ptr(q_window),
                                                _stream(stream)))


def sentencekv_decode_select(ctx, layer, q, input_token, sel_ids=None, sel_count=None, sel_tokens=None,
                             stream=None) -> None:
    """D1 (Eq. 2 + scores) + D2 (budgeted whole-sentence selection)."""
    _check(ctx, lib.sentencekv_decode_select(ctx, int(layer), _ptr(q), _ptr(input_token), _ptr(sel_ids),
                                             _ptr(sel_count), _ptr(sel_tokens), _stream(stream)))


def sentencekv_decode_attend(ctx, layer, q, out, stream=None) -> None:
    """D3 (gather) + D4 (Eq. 3 attention over the selected tokens) -> out fp32."""
    _check(ctx, lib.sentencekv_decode_attend(ctx, int(layer), _ptr(q), _ptr(out), _stream(stream)))


def sentencekv_decode_append(ctx, layer, k, v, input_token, stream=None) -> None:
    """NEXT-2: close the generated sentence that ended at the last token, append this token's k / v."""
    _check(ctx, lib.sentencekv_decode_append(ctx, int(layer), _ptr(k), _ptr(v), _ptr(input_token), _stream(stream)))


def sentencekv_decode_step(ctx, layer, q, input_token, out, sel_ids=None, sel_count=None, sel_tokens=None,
                           stream=None) -> None:
    """D1 + D2 + D3 + D4 in one call (fused select + attend; same results as select then attend)."""
    _check(ctx, lib.sentencekv_decode_step(ctx, int(layer), _ptr(q), _ptr(input_token), _ptr(out), _ptr(sel_ids),
                                           _ptr(sel_count), _ptr(sel_tokens), _stream(stream)))


# ------------------------------------------------------------------ convenience wrapper


class SentenceKV:
    """One ``skv_ctx`` plus shape bookkeeping.  All tensors are shard-local (see the header)."""

    def __init__(self, batch, layers, q_heads, kv_heads, head_dim, max_context, token_budget,
                 semantic_factor=2.0, residency=SKV_KV_DEVICE, device=0, kv_head_begin=0, kv_head_count=0,
                 batch_begin=0, batch_count=0, obs_window=0, bucket_mode=0, chunk_size=0, outlier_n=0.0,
                 query_mode=0, fill_mode=0, max_generated=0):
        self.cfg = sentencekv_config_default(
            batch=batch, layers=layers, q_heads=q_heads, kv_heads=kv_heads, head_dim=head_dim,
            max_context=max_context, token_budget=token_budget, semantic_factor=semantic_factor,
            residency=residency, device=device, kv_head_begin=kv_head_begin, kv_head_count=kv_head_count,
            batch_begin=batch_begin, batch_count=batch_count, obs_window=obs_window, bucket_mode=bucket_mode,
            chunk_size=chunk_size, outlier_n=outlier_n, query_mode=query_mode, fill_mode=fill_mode,
            max_generated=max_generated)
        self.quest = bucket_mode == SKV_BUCKETS_QUEST
        self.N = obs_window
        self.ctx = sentencekv_create(self.cfg)
        self.B = batch_count or (batch - batch_begin)
        self.G = kv_head_count or (kv_heads - kv_head_begin)
        self.grp = q_heads // kv_heads
        self.Hq = self.G * self.grp
        self.d = head_dim
        self.tau = token_budget
        self.r = semantic_factor
        self.device = torch.device("cuda", device)

    def close(self):
        if self.ctx:
            sentencekv_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prefill_compress(self, layer, K, V, token_ids=None, boundary_ids=None, q_window=None, stream=None):
        L = K.shape[2]
        sentencekv_prefill_compress(self.ctx, layer, token_ids, L, boundary_ids, K, V, self.r, self.tau, q_window,
                                    stream)

    def decode_select(self, layer, q, input_token, sel_ids=None, sel_count=None, sel_tokens=None, stream=None):
        sentencekv_decode_select(self.ctx, layer, q, input_token, sel_ids, sel_count, sel_tokens, stream)

    def decode_attend(self, layer, q, out, stream=None):
        sentencekv_decode_attend(self.ctx, layer, q, out, stream)

    def decode_append(self, layer, k, v, input_token, stream=None):
        """NEXT-2: this step's key / value [B][G][d] into the local segment (before the step's decode)."""
        sentencekv_decode_append(self.ctx, layer, k, v, input_token, stream)

    def set_output_peers(self, layer, rank, peer_out, peer_flag):
        """8(e) fused gather: peer_out / peer_flag = lists of device pointers (ints or tensors) of every rank."""
        world = len(peer_out)
        arr = lambda xs: (ctypes.c_void_p * world)(*[x.data_ptr() if isinstance(x, torch.Tensor) else int(x) for x in xs])
        _check(self.ctx, lib.sentencekv_set_output_peers(self.ctx, int(layer), world, int(rank), arr(peer_out),
                                                         arr(peer_flag)))

    def wait_outputs(self, layer, stream=None):
        _check(self.ctx, lib.sentencekv_wait_outputs(self.ctx, int(layer), _stream(stream)))

    def decode_step(self, layer, q, input_token, out, sel_ids=None, sel_count=None, sel_tokens=None, stream=None):
        sentencekv_decode_step(self.ctx, layer, q, input_token, out, sel_ids, sel_count, sel_tokens, stream)

    def sync(self):
        sentencekv_sync(self.ctx)

    # -- introspection --
    def sentence_counts(self):
        arr = (ctypes.c_int32 * self.B)()
        _check(self.ctx, lib.sentencekv_sentence_counts(self.ctx, arr))
        return list(arr)

    def capacity(self) -> int:
        return int(lib.sentencekv_sentence_capacity(self.ctx))

    def offsets(self, stream=None):
        S = self.capacity()
        out = torch.empty((self.B, S + 1), dtype=torch.int32, device=self.device)
        _check(self.ctx, lib.sentencekv_copy_offsets(self.ctx, _ptr(out), _stream(stream)))
        return out

    def embeddings(self, layer, stream=None):
        """[B][G][S_max][d] Eq. 1 means, or (Quest) [B][G][S_max][2][d] page (min, max) keys."""
        S = self.capacity()
        shape = (self.B, self.G, S, 2, self.d) if self.quest else (self.B, self.G, S, self.d)
        out = torch.empty(shape, dtype=torch.bfloat16, device=self.device)
        _check(self.ctx, lib.sentencekv_copy_embeddings(self.ctx, layer, _ptr(out), _stream(stream)))
        return out

    def scores(self, layer, stream=None):
        S = self.capacity()
        out = torch.empty((self.B, self.G, S), dtype=torch.float32, device=self.device)
        _check(self.ctx, lib.sentencekv_copy_scores(self.ctx, layer, _ptr(out), _stream(stream)))
        return out

    def host_fetch_bytes(self, layer) -> int:
        """Host residency ledger: K/V bytes fetched from host memory by the decode steps of `layer`."""
        v = ctypes.c_uint64()
        _check(self.ctx, lib.sentencekv_host_fetch_bytes(self.ctx, int(layer), ctypes.byref(v)))
        return int(v.value)

    def launch_count(self) -> int:
        return int(lib.sentencekv_launch_count(self.ctx))

    # NEXT-1 retention (obs_window > 0)
    def retained_tokens(self, layer) -> int:
        return int(lib.sentencekv_retained_tokens(self.ctx, int(layer)))

    def importance(self, layer, L, stream=None):
        """alpha fp32 [B][L - N] of the layer's prefill."""
        out = torch.empty((self.B, L - self.N), dtype=torch.float32, device=self.device)
        _check(self.ctx, lib.sentencekv_copy_importance(self.ctx, int(layer), _ptr(out), _stream(stream)))
        return out

    def retained(self, layer, stream=None):
        """(keep [B][m] token ids, bucket offsets [B][m+1], bucket sentence ids [B][m], buckets [B])."""
        m = self.retained_tokens(layer)
        keep = torch.empty((self.B, m), dtype=torch.int32, device=self.device)
        off = torch.empty((self.B, m + 1), dtype=torch.int32, device=self.device)
        sid = torch.empty((self.B, m), dtype=torch.int32, device=self.device)
        S = torch.empty((self.B,), dtype=torch.int32, device=self.device)
        _check(self.ctx, lib.sentencekv_copy_retained(self.ctx, int(layer), _ptr(keep), _ptr(off), _ptr(sid), _ptr(S),
                                                      _stream(stream)))
        return keep, off, sid, S

    KERNELS = ("segment", "compress", "score", "select", "attend", "retain", "step", "offload", "append")

    def set_profiling(self, on: bool):
        _check(self.ctx, lib.sentencekv_set_profiling(self.ctx, 1 if on else 0))

    def set_band_log2(self, log2: int):
        """Selection band width of decode_step (tuning; results are exact for any value)."""
        _check(self.ctx, lib.sentencekv_set_band_log2(self.ctx, int(log2)))

    def profile_read(self):
        """{kernel: (total_ms, launches)} of the profiled launches since the last read."""
        ms = (ctypes.c_double * len(self.KERNELS))()
        n = (ctypes.c_int64 * len(self.KERNELS))()
        _check(self.ctx, lib.sentencekv_profile_read(self.ctx, ms, n))
        return {k: (ms[i], n[i]) for i, k in enumerate(self.KERNELS)}
