/*
 * tkv.h — C ABI of the TableCache B200 online path (libtkv.so).
 *
 * Plain pointers and sizes only; every function returns a status (0 = ok) and never throws.
 * status = 1 + tablekv::Errc for the reference's error taxonomy (proj/include/tablekv/errors.hpp:9-28),
 * TKV_E_CUDA for CUDA failures, TKV_E_INVALID for bad arguments, TKV_E_INTERNAL otherwise;
 * tkv_last_error() returns the thread-local message of the last failure.
 *
 * The reference (proj/, C++20) has no FFI: its boundary is the C++ API in proj/include/tablekv.
 * Each entry point below names the reference interface it replaces; the headers under
 * include/tablekv/ are the source-level drop-in of the same API for C++ callers.
 */
#ifndef TKV_H_
#define TKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TKV_OK 0
#define TKV_E_CUDA 100
#define TKV_E_INVALID 101
#define TKV_E_INTERNAL 102

/* ---- errors / memory ------------------------------------------------------------------ */
int tkv_version(void);
/* copies the last error message of this thread into buf (NUL-terminated); returns its length */
size_t tkv_last_error(char* buf, size_t cap);
/* name of a status: "ok", "DanglingForeignKey" ... (errors.cpp:5-27), "CudaError", ... */
const char* tkv_status_name(int status);
/* frees strings returned through char** out-parameters */
void tkv_free(void* p);

/* ---- engine: corpus -> plan -> tokenizer -> trie (engine.cpp:16-52) -------------------- */
typedef struct tkv_engine tkv_engine;
/* replaces build_engine(EngineOptions{schema_path, topo_mode}) (engine.hpp:49) */
int tkv_engine_create(const char* schema_path, int break_cycles, tkv_engine** out);
/* same from the corpus JSON text (parse_schema_corpus, schema.hpp:75) */
int tkv_engine_create_json(const char* corpus_json, int break_cycles, tkv_engine** out);
void tkv_engine_destroy(tkv_engine* e);
/* JSON: vocab_size, vocab_hash, topo_order, removed_edges, groups[{tables,offsets}], group_of,
 * local_offset, table_tokens, serialized, edges, manifest */
int tkv_engine_info_json(const tkv_engine* e, char** json_out);
/* replaces analyze_query + assembly_order (engine.hpp:68-73): JSON tokens, spans[[id,s,e]],
 * match_order, remainder, assembly_order, record_tables */
int tkv_analyze_json(const tkv_engine* e, const char* query_id, const char* text, char** json_out);
/* replaces check_manifest (engine.hpp:58) */
int tkv_check_manifest(const tkv_engine* e, const char* cache_dir);
/* replaces run_workload (engine.hpp:87): the simulated SimReport::to_json() of a workload file */
int tkv_run_workload_json(const tkv_engine* e, const char* workload_path, const char* options_json, const char* kv_dir,
                          char** report_json);

/* ---- Table Trie (trie.hpp:34-64) ------------------------------------------------------ */
typedef struct tkv_trie tkv_trie;
int tkv_trie_create(tkv_trie** out);
void tkv_trie_destroy(tkv_trie* t);
int tkv_trie_insert(tkv_trie* t, const int32_t* tokens, size_t n, int table_id, uint64_t handle);
int tkv_trie_query(const tkv_trie* t, const int32_t* tokens, size_t n, size_t start, int* found, size_t* next,
                   int* table_id, uint64_t* handle);
/* spans_out: 3 int64 per span {table_id, start, end}; *n_spans = count (also when cap is short) */
int tkv_trie_match_all(const tkv_trie* t, const int32_t* tokens, size_t n, int64_t* spans_out, size_t cap,
                       size_t* n_spans, uint64_t* node_visits);

/* ---- reranking (rerank.hpp:22-44) ------------------------------------------------------ */
/* inc: [n][words] packed incidence bitsets; perm_out: n indices; threads 0 = auto */
int tkv_rerank(const uint64_t* inc, size_t n, size_t words, uint64_t seed, int fixed_first, int threads,
               uint64_t* perm_out);
/* the same permutation computed on GPU `device` (one thread-block cluster runs the greedy chain over
 * the distinct table sets; bit-exact) */
int tkv_rerank_device(int device, const uint64_t* inc, size_t n, size_t words, uint64_t seed, int fixed_first,
                      uint64_t* perm);
/* the calling thread's last tkv_rerank_device: out = {host class reduction ms, chain kernel ms (CUDA
 * events), whole call ms, distinct table sets, cluster CTAs (0: the compact single-CTA chain)} */
int tkv_rerank_device_stats(double* out, int n);

/* ---- fast-tier policy bookkeeping (tiered_cache.hpp:69-113) over a metadata slow tier --- */
typedef struct tkv_cache tkv_cache;
/* policy: 0 lru, 1 fifo, 2 lfu */
int tkv_cache_create(size_t capacity, int policy, const int32_t* token_counts, size_t n_tables, tkv_cache** out);
void tkv_cache_destroy(tkv_cache* c);
int tkv_cache_get(tkv_cache* c, int table_id, int* hit, int* evicted);
int tkv_cache_prefetch(tkv_cache* c, const int32_t* ids, size_t n, int32_t* admitted, size_t* n_admitted);
int tkv_cache_evict_candidate(const tkv_cache* c, int* table_id);
/* counters = {hits, misses, swaps, prefetch_loads}; residents sorted */
int tkv_cache_state(const tkv_cache* c, uint64_t counters[4], int32_t* residents, size_t cap, size_t* n_residents);

/* ---- pipeline (pipeline.hpp:54-102) ----------------------------------------------------- */
/* input JSON {token_counts, queries:[{id,tables,query_tokens}], runs:[{name, rerank_on, pipeline_on,
 * capacity, policy, b_c, b_m, seed, anchor, cost:{...}}]} -> per run {order, plan, trace, report,
 * report_overlapped, report_serial, final_residents} (schedule + build_trace + simulate + run_batch) */
int tkv_run_batch_json(const char* input_json, char** output_json);

/* ---- device model (model.hpp + attention.hpp:207-414 on the GPU) ------------------------ */
typedef struct tkv_model tkv_model;
typedef struct {
    int num_layers, num_heads, num_kv_heads, head_dim, ffn_dim, vocab_size;
    double rotary_base;
    uint64_t weight_seed;
    int mlp;   /* 0 SiLU (reference), 1 SwiGLU */
    int norm;  /* 0 LayerNorm w/o affine (reference), 1 RMSNorm */
    int dtype; /* 0 f32 reference-precision kernels, 1 bf16 tensor-core kernels, 2 f64 reference */
} tkv_model_config;
int tkv_model_create(int device, const tkv_model_config* cfg, tkv_model** out);
void tkv_model_destroy(tkv_model* m);
/* attention kernel of bf16 models: 0 tcgen05 where supported (head_dim 128), 1 mma.sync */
int tkv_model_set_attention(tkv_model* m, int impl);
/* which: 0 embedding [vocab][hidden], 1 head [vocab(_padded for bf16)][hidden]; raw model-dtype bytes */
int tkv_model_weights(tkv_model* m, int which, void* host_out, size_t bytes);
/* One sequence through the device forward with host buffers (the parity wrappers of prefill /
 * query_attend / encode_group, attention.hpp:210-414). tokens/positions/groups: n entries.
 * mode 0: own rows attend all n_ctx cached rows + causal own (ctx_k/ctx_v: [L][n_ctx][kv_dim],
 * rotated, model dtype); mode 1: block-causal by group id (BlockMask::allows), no ctx.
 * Outputs (nullable): hidden [n][hidden] (f32 for bf16 models, else model dtype),
 * kraw/v [L][n][kv_dim] (model dtype), logits [vocab_padded] f32 + argmax of the last row. */
int tkv_model_forward(tkv_model* m, const int32_t* tokens, const int32_t* positions, const int32_t* groups, int n,
                      int mode, const void* ctx_k, const void* ctx_v, int n_ctx, void* hidden_out, void* kraw_out,
                      void* v_out, float* logits_out, int32_t* argmax_out);

/* ---- table store: pinned arena (slow tier) + paged HBM pool (fast tier) + executor --------- */
typedef struct tkv_store tkv_store;
int tkv_store_create(tkv_model* m, size_t page_bytes, int n_pages, tkv_store** out);
void tkv_store_destroy(tkv_store* s);
/* SlowTier::load payload (table_kv.hpp:45-48 layout, no header): dtype 0 f32, 1 bf16 */
int tkv_store_put(tkv_store* s, int table_id, int tokens, int local_offset, int dtype, const void* payload);
/* a reference .kv file (FileSlowTier::load, tiered_cache.cpp:49-59) straight into the arena */
int tkv_store_load_kv_file(tkv_store* s, const char* path, int* table_id);
/* a precompute directory (<id>.kv f32 reference files and/or <id>.kvb bf16 images) straight into
 * the pinned arena with `threads` readers (0: 8); e (nullable) checks manifest.json first
 * (check_manifest, engine.cpp:114-131). Tables already in the arena are skipped. */
int tkv_store_load_dir(tkv_store* s, const char* dir, const tkv_engine* e, int threads, int* n_loaded);
/* offline encode of every group on the GPU (precompute_corpus, engine.cpp:83-112) into the arena;
 * out_dir (nullable) also gets <id>.kv files (f32 models: the reference format) + manifest.json */
int tkv_store_precompute(tkv_store* s, const tkv_engine* e, const char* out_dir);
/* stats of the last precompute into out[0..n): groups, tables, tokens, forwards, device ms (encode
 * forwards + D2H into the arena), GEMM ms, GEMM flops, attention ms, kernel launches (the timed
 * fields need timed_next = 1 set before that precompute: CUDA events around each launch) */
int tkv_store_precompute_stats(const tkv_store* s, int timed_next, double* out, int n);
/* copy a table into pool pages (one miss), read the landed bytes back (bytes-exact check) */
int tkv_store_fetch(tkv_store* s, int table_id, int copy_engine, void* host_out, size_t bytes);
/* assemble() on the GPU (attention.hpp:300-362): k_out/v_out [L][total][kv_dim] (dense, row stride
 * total) in the model's serving dtype (f32 for f32 models, bf16 otherwise), each buffer holding
 * cap_tokens rows per layer at least; *total_tokens gets the prefix length (also on the
 * too-small error, so a caller can size and retry; null outputs = length only) */
int tkv_store_assemble(tkv_store* s, const int32_t* tables, int n_tables, size_t cap_tokens, void* k_out, void* v_out,
                       int* total_tokens);
/* arena footprint */
int tkv_store_info(const tkv_store* s, size_t* tables, size_t* arena_bytes, size_t* free_pages);

typedef struct {
    int rerank_on, pipeline_on;
    size_t capacity;
    int policy;  /* 0 lru, 1 fifo, 2 lfu */
    int b_c, b_m;
    uint64_t seed;
    int fixed_anchor;
    double compute_per_token, load_per_token, switch_overhead;
    int copy_engine;   /* 0 DMA copy engines, 1 SM 16-byte vector copy kernel */
    int sm_copy_ctas;
    int nocache;       /* 1: the no-cache baseline (block-masked full prefill, same kernels) */
    int time_kernels;  /* per-GEMM CUDA events (roofline) */
    int peer_fetch;    /* 1: misses predicted resident on an attached peer GPU are copied over NVLink */
    int peer_ctas;     /* CTAs per peer-fetch copy */
} tkv_serve_options;
void tkv_serve_options_default(tkv_serve_options* o);

/* The online path for a batch (run_batch, pipeline.cpp:310-342, executed for real): queries i has
 * tables[table_off[i]:table_off[i+1]] in assembly order and suffix[suffix_off[i]:...] remainder tokens.
 * logits_out (nullable): [n][vocab_padded] f32 in SERVED order. result_json: order, ttft_ms, argmax,
 * window_of, window_end_ms, trace, counters, h2d_bytes, copy_busy_ms, makespan_ms, host_ms, launches,
 * gemm_ms/gemm_flops/gather_ms/attn_ms (time_kernels). */
int tkv_serve(tkv_store* s, size_t n, const int64_t* table_off, const int32_t* tables, const int64_t* suffix_off,
              const int32_t* suffix, const tkv_serve_options* o, float* logits_out, char** result_json);
/* the same from prompt text: analyze_query + assembly_order on the host, then tkv_serve */
int tkv_serve_text(tkv_store* s, const tkv_engine* e, size_t n, const char* const* ids, const char* const* texts,
                   const tkv_serve_options* o, float* logits_out, char** result_json);
/* binds corpus token ids + group ids (needed by the no-cache baseline) */
int tkv_store_bind_engine(tkv_store* s, const tkv_engine* e);

/* ---- NVLink peer KV fetch (no reference counterpart: the reference is one
 * process). A miss whose table is resident in a peer GPU's pool is copied from that pool over
 * NVLink instead of from the host arena; it changes the SOURCE of a miss, never the trace.
 * export: the opaque IPC blob of this store (pool slab + residency directory), *n = its size;
 * dir_entries = table-id capacity of the directory (0: max arena table id + 1).
 * attach: the blobs of the n peers (peer slot i = blobs[i]); once per store.
 * plan: peer slot's upcoming batch (tables per query in assembly order, suffix lengths) for the
 * host-side residency prediction that routes misses; serve() with peer_fetch = 1 uses it.
 * publish/unpublish: hold a table resident in this store's pool and visible to peers (tests,
 * static sharing). fetch: copy a table into fresh pages from the first peer holding it (host
 * arena per CTA otherwise) and read the landed bytes back; *peer_bytes = bytes served by peers. */
int tkv_store_peer_export(tkv_store* s, int dir_entries, void* blob_out, size_t cap, size_t* n);
int tkv_store_peer_attach(tkv_store* s, int n, const void* const* blobs, const size_t* sizes);
int tkv_store_peer_plan(tkv_store* s, int slot, size_t n, const int64_t* table_off, const int32_t* tables,
                        const int32_t* suffix_len);
int tkv_store_peer_publish(tkv_store* s, int table_id);
int tkv_store_peer_unpublish(tkv_store* s, int table_id);
int tkv_store_peer_fetch(tkv_store* s, int table_id, void* host_out, size_t bytes, uint64_t* peer_bytes);

/* ---- measurement helpers ---------------------------------------------------------------- */
/* pinned H2D copy peak over `bytes`, best of `reps` (GB/s) */
int tkv_measure_h2d(int device, size_t bytes, int reps, double* gbs);
/* bf16 GEMM through the tcgen05 kernel (epilogue 0 store_bf16, 1 store_f32): A [M][K], B [N][K] host
 * bf16 bits, C host; simt=1 runs the SIMT reference kernel instead; ms_out = event time */
int tkv_debug_gemm(int M, int N, int K, const uint16_t* A, const uint16_t* B, int epilogue, int simt, void* C,
                   double* ms_out);

#ifdef __cplusplus
}
#endif

#endif /* TKV_H_ */
