"""ctypes binding of libtkv.so (include/tkv.h) — the host-side mirror of the reference API.

Names follow the reference (proj/include/tablekv): Engine (build_engine / analyze_query /
assembly_order), Trie (TableTrie), rerank, Cache (TieredCache), run_batch_json (schedule +
build_trace + simulate + run_batch), and the device side: Model (prefill / query_attend /
encode_group on the GPU) and Store (pinned arena + paged HBM pool + the serving executor).
Errors come back as TkvError carrying the reference's error name (errors.cpp:5-27).
There is no fallback: if the library is missing, import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TKV_LIB") or os.path.join(_HERE, "lib", "libtkv.so")  # TKV_LIB: A/B builds only

if not os.path.exists(LIB_PATH):
    raise ImportError("libtkv.so not built: run `make -C paper_2601_08743_b200` (or __graft_entry__.build())")
_lib = C.CDLL(LIB_PATH)

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)
_fp = C.POINTER(C.c_float)
_vp = C.c_void_p


class TkvError(RuntimeError):
    def __init__(self, status, name, msg):
        super().__init__("%s (%d): %s" % (name, status, msg))
        self.status, self.name, self.msg = status, name, msg


class tkv_model_config(C.Structure):
    _fields_ = [("num_layers", C.c_int), ("num_heads", C.c_int), ("num_kv_heads", C.c_int), ("head_dim", C.c_int),
                ("ffn_dim", C.c_int), ("vocab_size", C.c_int), ("rotary_base", C.c_double), ("weight_seed", C.c_uint64),
                ("mlp", C.c_int), ("norm", C.c_int), ("dtype", C.c_int)]


class tkv_serve_options(C.Structure):
    _fields_ = [("rerank_on", C.c_int), ("pipeline_on", C.c_int), ("capacity", C.c_size_t), ("policy", C.c_int),
                ("b_c", C.c_int), ("b_m", C.c_int), ("seed", C.c_uint64), ("fixed_anchor", C.c_int),
                ("compute_per_token", C.c_double), ("load_per_token", C.c_double), ("switch_overhead", C.c_double),
                ("copy_engine", C.c_int), ("sm_copy_ctas", C.c_int), ("nocache", C.c_int), ("time_kernels", C.c_int),
                ("peer_fetch", C.c_int), ("peer_ctas", C.c_int)]


def _sig(name, *args, res=C.c_int):
    f = getattr(_lib, name)
    f.argtypes = list(args)
    f.restype = res
    return f


_sig("tkv_last_error", C.c_char_p, C.c_size_t, res=C.c_size_t)
_sig("tkv_status_name", C.c_int, res=C.c_char_p)
_sig("tkv_free", _vp, res=None)
_sig("tkv_engine_create", C.c_char_p, C.c_int, C.POINTER(_vp))
_sig("tkv_engine_create_json", C.c_char_p, C.c_int, C.POINTER(_vp))
_sig("tkv_engine_destroy", _vp, res=None)
_sig("tkv_engine_info_json", _vp, C.POINTER(_vp))
_sig("tkv_analyze_json", _vp, C.c_char_p, C.c_char_p, C.POINTER(_vp))
_sig("tkv_check_manifest", _vp, C.c_char_p)
_sig("tkv_run_workload_json", _vp, C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(_vp))
_sig("tkv_trie_create", C.POINTER(_vp))
_sig("tkv_trie_destroy", _vp, res=None)
_sig("tkv_trie_insert", _vp, _i32p, C.c_size_t, C.c_int, C.c_uint64)
_sig("tkv_trie_query", _vp, _i32p, C.c_size_t, C.c_size_t, C.POINTER(C.c_int), C.POINTER(C.c_size_t),
     C.POINTER(C.c_int), _u64p)
_sig("tkv_trie_match_all", _vp, _i32p, C.c_size_t, _i64p, C.c_size_t, C.POINTER(C.c_size_t), _u64p)
_sig("tkv_rerank", _u64p, C.c_size_t, C.c_size_t, C.c_uint64, C.c_int, C.c_int, _u64p)
_sig("tkv_rerank_device", C.c_int, _u64p, C.c_size_t, C.c_size_t, C.c_uint64, C.c_int, _u64p)
_sig("tkv_rerank_device_stats", C.POINTER(C.c_double), C.c_int)
_sig("tkv_cache_create", C.c_size_t, C.c_int, _i32p, C.c_size_t, C.POINTER(_vp))
_sig("tkv_cache_destroy", _vp, res=None)
_sig("tkv_cache_get", _vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int))
_sig("tkv_cache_prefetch", _vp, _i32p, C.c_size_t, _i32p, C.POINTER(C.c_size_t))
_sig("tkv_cache_evict_candidate", _vp, C.POINTER(C.c_int))
_sig("tkv_cache_state", _vp, _u64p, _i32p, C.c_size_t, C.POINTER(C.c_size_t))
_sig("tkv_run_batch_json", C.c_char_p, C.POINTER(_vp))
_sig("tkv_model_create", C.c_int, C.POINTER(tkv_model_config), C.POINTER(_vp))
_sig("tkv_model_destroy", _vp, res=None)
_sig("tkv_model_weights", _vp, C.c_int, _vp, C.c_size_t)
_sig("tkv_model_set_attention", _vp, C.c_int)
_sig("tkv_model_forward", _vp, _i32p, _i32p, _i32p, C.c_int, C.c_int, _vp, _vp, C.c_int, _vp, _vp, _vp, _fp, _i32p)
_sig("tkv_store_create", _vp, C.c_size_t, C.c_int, C.POINTER(_vp))
_sig("tkv_store_destroy", _vp, res=None)
_sig("tkv_store_put", _vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp)
_sig("tkv_store_load_kv_file", _vp, C.c_char_p, C.POINTER(C.c_int))
_sig("tkv_store_load_dir", _vp, C.c_char_p, _vp, C.c_int, C.POINTER(C.c_int))
_sig("tkv_store_precompute", _vp, _vp, C.c_char_p)
_sig("tkv_store_precompute_stats", _vp, C.c_int, C.POINTER(C.c_double), C.c_int)
_sig("tkv_store_fetch", _vp, C.c_int, C.c_int, _vp, C.c_size_t)
_sig("tkv_store_assemble", _vp, _i32p, C.c_int, C.c_size_t, _vp, _vp, C.POINTER(C.c_int))
_sig("tkv_store_info", _vp, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t))
_sig("tkv_store_bind_engine", _vp, _vp)
_sig("tkv_serve_options_default", C.POINTER(tkv_serve_options), res=None)
_sig("tkv_store_peer_export", _vp, C.c_int, _vp, C.c_size_t, C.POINTER(C.c_size_t))
_sig("tkv_store_peer_attach", _vp, C.c_int, C.POINTER(_vp), C.POINTER(C.c_size_t))
_sig("tkv_store_peer_plan", _vp, C.c_int, C.c_size_t, _i64p, _i32p, _i32p)
_sig("tkv_store_peer_publish", _vp, C.c_int)
_sig("tkv_store_peer_unpublish", _vp, C.c_int)
_sig("tkv_store_peer_fetch", _vp, C.c_int, _vp, C.c_size_t, _u64p)
_sig("tkv_serve", _vp, C.c_size_t, _i64p, _i32p, _i64p, _i32p, C.POINTER(tkv_serve_options), _fp, C.POINTER(_vp))
_sig("tkv_serve_text", _vp, _vp, C.c_size_t, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p),
     C.POINTER(tkv_serve_options), _fp, C.POINTER(_vp))
_sig("tkv_measure_h2d", C.c_int, C.c_size_t, C.c_int, C.POINTER(C.c_double))
_sig("tkv_debug_gemm", C.c_int, C.c_int, C.c_int, _vp, _vp, C.c_int, C.c_int, _vp, C.POINTER(C.c_double))

# every symbol the header declares (checked by the CPU tests)
EXPORTED = [l.split("(")[0].split()[-1].lstrip("*")
            for l in open(os.path.join(os.path.dirname(_HERE), "include", "tkv.h"))
            if l.strip().startswith(("int tkv_", "void tkv_", "size_t tkv_", "const char* tkv_"))]


def _check(rc):
    if rc != 0:
        buf = C.create_string_buffer(4096)
        _lib.tkv_last_error(buf, 4096)
        raise TkvError(rc, _lib.tkv_status_name(rc).decode(), buf.value.decode(errors="replace"))


def _take_string(p):
    s = C.cast(p, C.c_char_p).value.decode()
    _lib.tkv_free(p)
    return s


def _arr(a, dtype):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


def _ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


def status_name(rc):
    return _lib.tkv_status_name(rc).decode()


# ----------------------------------------------------------------------------- engine

class Engine:
    """build_engine (engine.cpp:16-52) over a schema corpus file or JSON text."""

    def __init__(self, schema_path=None, corpus_json=None, break_cycles=False):
        h = _vp()
        if schema_path is not None:
            _check(_lib.tkv_engine_create(schema_path.encode(), int(break_cycles), C.byref(h)))
        else:
            _check(_lib.tkv_engine_create_json(corpus_json.encode(), int(break_cycles), C.byref(h)))
        self._h = h
        out = _vp()
        _check(_lib.tkv_engine_info_json(self._h, C.byref(out)))
        self.info = json.loads(_take_string(out))

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.tkv_engine_destroy(self._h)
            self._h = None

    def analyze(self, text, query_id=""):
        out = _vp()
        _check(_lib.tkv_analyze_json(self._h, query_id.encode(), text.encode(), C.byref(out)))
        return json.loads(_take_string(out))

    def check_manifest(self, cache_dir):
        _check(_lib.tkv_check_manifest(self._h, cache_dir.encode()))

    def run_workload(self, workload_path, options=None, kv_dir=None):
        out = _vp()
        _check(_lib.tkv_run_workload_json(self._h, workload_path.encode(), json.dumps(options or {}).encode(),
                                          kv_dir.encode() if kv_dir else None, C.byref(out)))
        return json.loads(_take_string(out))


class Trie:
    """TableTrie (trie.hpp:34-64)."""

    def __init__(self):
        h = _vp()
        _check(_lib.tkv_trie_create(C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.tkv_trie_destroy(self._h)
            self._h = None

    def insert(self, tokens, table_id, handle=None):
        t = _arr(tokens, np.int32)
        _check(_lib.tkv_trie_insert(self._h, _ptr(t, C.c_int32), len(t), table_id,
                                    table_id if handle is None else handle))

    def query(self, tokens, start):
        t = _arr(tokens, np.int32)
        f, n, tid, hd = C.c_int(), C.c_size_t(), C.c_int(), C.c_uint64()
        _check(_lib.tkv_trie_query(self._h, _ptr(t, C.c_int32), len(t), start, C.byref(f), C.byref(n), C.byref(tid),
                                   C.byref(hd)))
        return bool(f.value), n.value, tid.value

    def match_all(self, tokens):
        t = _arr(tokens, np.int32)
        cap = max(1, len(t))
        out = np.zeros(3 * cap, np.int64)
        n, visits = C.c_size_t(), C.c_uint64()
        _check(_lib.tkv_trie_match_all(self._h, _ptr(t, C.c_int32), len(t), _ptr(out, C.c_int64), cap, C.byref(n),
                                       C.byref(visits)))
        return [tuple(int(x) for x in out[3 * i:3 * i + 3]) for i in range(n.value)], visits.value


def pack_incidence(table_sets, n_bits):
    words = max(1, (n_bits + 63) // 64)
    inc = np.zeros((len(table_sets), words), np.uint64)
    lens = np.fromiter((len(ts) for ts in table_sets), np.int64, len(table_sets))
    if lens.sum():
        ids = np.fromiter((t for ts in table_sets for t in ts), np.int64, int(lens.sum()))
        if ids.min() < 0 or ids.max() >= n_bits:
            raise ValueError("table id out of range")
        rows = np.repeat(np.arange(len(table_sets)), lens)
        np.bitwise_or.at(inc, (rows, ids >> 6), np.left_shift(np.uint64(1), (ids & 63).astype(np.uint64)))
    return inc


def rerank(table_sets, n_bits, seed=1, mode="seeded", threads=0):
    """rerank (rerank.cpp:55-94) over per-query table sets."""
    inc = pack_incidence(table_sets, n_bits)
    perm = np.zeros(len(table_sets), np.uint64)
    _check(_lib.tkv_rerank(_ptr(inc, C.c_uint64), inc.shape[0], inc.shape[1], seed, int(mode == "fixed_first"), threads,
                           _ptr(perm, C.c_uint64)))
    return [int(x) for x in perm]


def rerank_device(table_sets, n_bits, seed=1, mode="seeded", device=0):
    """rerank on the GPU: the same permutation as rerank() (rerank.cpp:55-94)."""
    inc = pack_incidence(table_sets, n_bits)
    perm = np.zeros(len(table_sets), np.uint64)
    _check(_lib.tkv_rerank_device(device, _ptr(inc, C.c_uint64), inc.shape[0], inc.shape[1], seed,
                                  int(mode == "fixed_first"), _ptr(perm, C.c_uint64)))
    return [int(x) for x in perm]


def rerank_device_stats():
    """The calling thread's last rerank_device: host class reduction ms, chain kernel ms (CUDA events),
    whole call ms, distinct table sets, cluster CTAs."""
    v = (C.c_double * 5)()
    _check(_lib.tkv_rerank_device_stats(v, 5))
    return dict(zip(("classes_ms", "kernel_ms", "call_ms", "classes", "cluster"), list(v)))


POLICIES = {"lru": 0, "fifo": 1, "lfu": 2}


class Cache:
    """TieredCache (tiered_cache.hpp:69-113) over a metadata-only slow tier."""

    def __init__(self, capacity, policy, token_counts):
        tc = _arr(token_counts, np.int32)
        h = _vp()
        _check(_lib.tkv_cache_create(capacity, POLICIES[policy], _ptr(tc, C.c_int32), len(tc), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.tkv_cache_destroy(self._h)
            self._h = None

    def get(self, table_id):
        hit, ev = C.c_int(), C.c_int()
        _check(_lib.tkv_cache_get(self._h, table_id, C.byref(hit), C.byref(ev)))
        return bool(hit.value), ev.value

    def prefetch(self, ids):
        a = _arr(ids, np.int32)
        out = np.zeros(max(1, len(a)), np.int32)
        n = C.c_size_t()
        _check(_lib.tkv_cache_prefetch(self._h, _ptr(a, C.c_int32), len(a), _ptr(out, C.c_int32), C.byref(n)))
        return [int(x) for x in out[:n.value]]

    def evict_candidate(self):
        v = C.c_int()
        _check(_lib.tkv_cache_evict_candidate(self._h, C.byref(v)))
        return v.value

    def state(self):
        cnt = np.zeros(4, np.uint64)
        res = np.zeros(4096, np.int32)
        n = C.c_size_t()
        _check(_lib.tkv_cache_state(self._h, _ptr(cnt, C.c_uint64), _ptr(res, C.c_int32), 4096, C.byref(n)))
        return [int(x) for x in cnt], [int(x) for x in res[:n.value]]


def run_batch_json(payload):
    """schedule + build_trace + simulate + run_batch for each run in the payload."""
    out = _vp()
    _check(_lib.tkv_run_batch_json(json.dumps(payload).encode(), C.byref(out)))
    return json.loads(_take_string(out))


# ----------------------------------------------------------------------------- device

DTYPES = {"f32": 0, "bf16": 1, "f64": 2}
NP_DTYPES = {0: np.float32, 1: np.uint16, 2: np.float64}


class Model:
    """Device model: weights from the counter hash, prefill / query_attend / encode_group."""

    def __init__(self, num_layers=2, num_heads=4, head_dim=16, vocab_size=330, num_kv_heads=0, ffn_dim=0,
                 rotary_base=10000.0, weight_seed=1, mlp="silu", norm="ln", dtype="f32", device=0):
        cfg = tkv_model_config(num_layers, num_heads, num_kv_heads or num_heads, head_dim,
                               ffn_dim or 4 * num_heads * head_dim, vocab_size, rotary_base, weight_seed,
                               int(mlp == "swiglu"), int(norm == "rms"), DTYPES[dtype])
        self.cfg = cfg
        self.dtype = DTYPES[dtype]
        self.hidden = num_heads * head_dim
        self.kv_dim = cfg.num_kv_heads * head_dim
        self.vocab_padded = (vocab_size + 255) // 256 * 256
        h = _vp()
        _check(_lib.tkv_model_create(device, C.byref(cfg), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _lib.tkv_model_destroy(self._h)
            self._h = None

    __del__ = close

    def set_attention(self, impl):
        """0 = tcgen05 attention where supported (head_dim 128), 1 = mma.sync kernel."""
        _check(_lib.tkv_model_set_attention(self._h, {"tc5": 0, "mma": 1}.get(impl, impl)))

    def weights(self, which):
        rows = self.cfg.vocab_size if (which == 0 or self.dtype != 1) else self.vocab_padded
        out = np.zeros((rows, self.hidden), NP_DTYPES[self.dtype])
        _check(_lib.tkv_model_weights(self._h, which, out.ctypes.data, out.nbytes))
        return out

    def forward(self, tokens, positions=None, groups=None, mode=0, ctx_k=None, ctx_v=None, want_kv=False,
                want_logits=True):
        """One sequence. mode 0: attends all ctx rows (ctx_k/v [L][n_ctx][kv_dim]) + causal own;
        mode 1: block-causal by group id. Returns dict(hidden, kraw, v, logits, argmax)."""
        t = _arr(tokens, np.int32)
        n = len(t)
        p = _arr(positions, np.int32) if positions is not None else None
        g = _arr(groups, np.int32) if groups is not None else None
        edt = NP_DTYPES[self.dtype]
        L = self.cfg.num_layers
        ck = _arr(ctx_k, edt) if ctx_k is not None else None
        cv = _arr(ctx_v, edt) if ctx_v is not None else None
        n_ctx = 0 if ck is None else ck.shape[1]
        hidden = np.zeros((n, self.hidden), np.float32 if self.dtype == 1 else edt)
        kraw = np.zeros((L, n, self.kv_dim), edt) if want_kv else None
        v = np.zeros((L, n, self.kv_dim), edt) if want_kv else None
        logits = np.zeros(self.vocab_padded, np.float32) if want_logits else None
        am = np.zeros(1, np.int32) if want_logits else None
        _check(_lib.tkv_model_forward(self._h, _ptr(t, C.c_int32), _ptr(p, C.c_int32), _ptr(g, C.c_int32), n, mode,
                                      ck.ctypes.data if ck is not None else None,
                                      cv.ctypes.data if cv is not None else None, n_ctx, hidden.ctypes.data,
                                      kraw.ctypes.data if want_kv else None, v.ctypes.data if want_kv else None,
                                      _ptr(logits, C.c_float), _ptr(am, C.c_int32)))
        return {"hidden": hidden, "kraw": kraw, "v": v,
                "logits": logits[:self.cfg.vocab_size] if want_logits else None,
                "argmax": int(am[0]) if want_logits else None}


def serve_options(**kw):
    o = tkv_serve_options()
    _lib.tkv_serve_options_default(C.byref(o))
    pol = kw.pop("policy", None)
    if pol is not None:
        o.policy = POLICIES[pol] if isinstance(pol, str) else pol
    for k, v in kw.items():
        setattr(o, k, v)
    return o


class Store:
    """Pinned arena (slow tier) + paged HBM pool (fast tier) + the serving executor."""

    def __init__(self, model: Model, page_bytes=2 << 20, n_pages=256):
        h = _vp()
        _check(_lib.tkv_store_create(model._h, page_bytes, n_pages, C.byref(h)))
        self._h = h
        self.model = model

    def close(self):
        if getattr(self, "_h", None):
            _lib.tkv_store_destroy(self._h)
            self._h = None

    __del__ = close

    def put(self, table_id, tokens, local_offset, payload, dtype):
        a = np.ascontiguousarray(payload)
        _check(_lib.tkv_store_put(self._h, table_id, tokens, local_offset, DTYPES[dtype], a.ctypes.data))

    def load_kv_file(self, path):
        tid = C.c_int()
        _check(_lib.tkv_store_load_kv_file(self._h, path.encode(), C.byref(tid)))
        return tid.value

    def load_dir(self, path, engine=None, threads=0):
        """A precompute directory (.kv f32 / .kvb bf16) into the pinned arena; returns tables loaded."""
        n = C.c_int()
        _check(_lib.tkv_store_load_dir(self._h, path.encode(), engine._h if engine else None, threads, C.byref(n)))
        return n.value

    def precompute(self, engine: Engine, out_dir=None, timed=False):
        """Offline encode of every group on the GPU (batched block-causal forwards) into the arena;
        returns the encode stats (timed=True adds CUDA-event GEMM / attention times)."""
        _check(_lib.tkv_store_precompute_stats(self._h, int(timed), None, 0))
        _check(_lib.tkv_store_precompute(self._h, engine._h, out_dir.encode() if out_dir else None))
        v = (C.c_double * 9)()
        _check(_lib.tkv_store_precompute_stats(self._h, 0, v, 9))
        keys = ("groups", "tables", "tokens", "forwards", "device_ms", "gemm_ms", "gemm_flops", "attn_ms", "launches")
        return dict(zip(keys, list(v)))

    def bind_engine(self, engine: Engine):
        _check(_lib.tkv_store_bind_engine(self._h, engine._h))

    def fetch(self, table_id, nbytes, copy_engine=0):
        out = np.zeros(nbytes, np.uint8)
        _check(_lib.tkv_store_fetch(self._h, table_id, copy_engine, out.ctypes.data, nbytes))
        return out

    def assemble(self, tables, total_hint=None):
        """[L][total][kv_dim] rotated K and V of the tables concatenated in order (total_hint unused:
        the prefix length is asked first)."""
        L, kvd = self.model.cfg.num_layers, self.model.kv_dim
        edt = np.uint16 if self.model.dtype == 1 else np.float32
        t = _arr(tables, np.int32)
        total = C.c_int()
        _check(_lib.tkv_store_assemble(self._h, _ptr(t, C.c_int32), len(t), 0, None, None, C.byref(total)))
        n = max(1, total.value)
        k = np.zeros((L, n, kvd), edt)
        v = np.zeros_like(k)
        _check(_lib.tkv_store_assemble(self._h, _ptr(t, C.c_int32), len(t), n, k.ctypes.data, v.ctypes.data,
                                       C.byref(total)))
        return k[:, :total.value], v[:, :total.value]

    def info(self):
        a, b, c = C.c_size_t(), C.c_size_t(), C.c_size_t()
        _check(_lib.tkv_store_info(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return {"tables": a.value, "arena_bytes": b.value, "free_pages": c.value}

    def serve(self, queries, options=None, want_logits=False, **kw):
        """queries: list of (tables_in_assembly_order, suffix_tokens). Returns the result dict
        (+ 'logits' [n][vocab] in served order when asked)."""
        o = options or serve_options(**kw)
        toff = np.zeros(len(queries) + 1, np.int64)
        soff = np.zeros(len(queries) + 1, np.int64)
        for i, (ts, sx) in enumerate(queries):
            toff[i + 1] = toff[i] + len(ts)
            soff[i + 1] = soff[i] + len(sx)
        tabs = _arr([t for ts, _ in queries for t in ts] or [0], np.int32)
        suf = _arr([x for _, sx in queries for x in sx] or [0], np.int32)
        logits = np.zeros((len(queries), self.model.vocab_padded), np.float32) if want_logits else None
        out = _vp()
        _check(_lib.tkv_serve(self._h, len(queries), _ptr(toff, C.c_int64), _ptr(tabs, C.c_int32),
                              _ptr(soff, C.c_int64), _ptr(suf, C.c_int32), C.byref(o), _ptr(logits, C.c_float),
                              C.byref(out)))
        r = json.loads(_take_string(out))
        if want_logits:
            r["logits"] = logits[:, :self.model.cfg.vocab_size]
        return r

    # ---- NVLink peer KV fetch
    def peer_export(self, dir_entries=0) -> bytes:
        """This store's IPC blob (pool slab + residency directory) for the other ranks."""
        n = C.c_size_t()
        _check(_lib.tkv_store_peer_export(self._h, dir_entries, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _check(_lib.tkv_store_peer_export(self._h, dir_entries, C.cast(buf, _vp), n.value, C.byref(n)))
        return buf.raw[:n.value]

    def peer_attach(self, blobs):
        """blobs: the other ranks' peer_export() bytes; peer slot i = blobs[i]."""
        bufs = [C.create_string_buffer(b, len(b)) for b in blobs]
        arr = (_vp * max(1, len(bufs)))(*[C.cast(b, _vp) for b in bufs])
        sizes = (C.c_size_t * max(1, len(bufs)))(*[len(b) for b in blobs])
        _check(_lib.tkv_store_peer_attach(self._h, len(bufs), arr, sizes))

    def peer_plan(self, slot, queries):
        """queries: the peer's upcoming batch as (tables, suffix or suffix length) pairs."""
        toff = np.zeros(len(queries) + 1, np.int64)
        for i, (ts, _) in enumerate(queries):
            toff[i + 1] = toff[i] + len(ts)
        tabs = _arr([t for ts, _ in queries for t in ts] or [0], np.int32)
        sl = _arr([sx if isinstance(sx, int) else len(sx) for _, sx in queries] or [0], np.int32)
        _check(_lib.tkv_store_peer_plan(self._h, slot, len(queries), _ptr(toff, C.c_int64), _ptr(tabs, C.c_int32),
                                        _ptr(sl, C.c_int32)))

    def peer_publish(self, table_id):
        _check(_lib.tkv_store_peer_publish(self._h, table_id))

    def peer_unpublish(self, table_id):
        _check(_lib.tkv_store_peer_unpublish(self._h, table_id))

    def peer_fetch(self, table_id, nbytes):
        """(landed bytes, bytes that came from a peer)"""
        out = np.zeros(nbytes, np.uint8)
        pb = C.c_uint64()
        _check(_lib.tkv_store_peer_fetch(self._h, table_id, out.ctypes.data, nbytes, C.byref(pb)))
        return out, pb.value

    def serve_text(self, engine: Engine, texts, ids=None, options=None, want_logits=False, **kw):
        o = options or serve_options(**kw)
        n = len(texts)
        ids = ids or ["q%d" % i for i in range(n)]
        tarr = (C.c_char_p * n)(*[t.encode() for t in texts])
        iarr = (C.c_char_p * n)(*[i.encode() for i in ids])
        logits = np.zeros((n, self.model.vocab_padded), np.float32) if want_logits else None
        out = _vp()
        _check(_lib.tkv_serve_text(self._h, engine._h, n, iarr, tarr, C.byref(o), _ptr(logits, C.c_float),
                                   C.byref(out)))
        r = json.loads(_take_string(out))
        if want_logits:
            r["logits"] = logits[:, :self.model.cfg.vocab_size]
        return r


def measure_h2d(bytes_=256 << 20, reps=5, device=0):
    g = C.c_double()
    _check(_lib.tkv_measure_h2d(device, bytes_, reps, C.byref(g)))
    return g.value


def debug_gemm(A_bits, B_bits, epilogue=1, simt=0):
    A = np.ascontiguousarray(A_bits, dtype=np.uint16)
    B = np.ascontiguousarray(B_bits, dtype=np.uint16)
    M, K = A.shape
    N = B.shape[0]
    out = np.zeros((M, N), np.float32 if epilogue == 1 else np.uint16)
    ms = C.c_double()
    _check(_lib.tkv_debug_gemm(M, N, K, A.ctypes.data, B.ctypes.data, epilogue, int(simt), out.ctypes.data,
                               C.byref(ms)))
    return out, ms.value
