/* nmt.h - C ABI of libnmt.so: batched GPU querying of an attention-based encoder-decoder
 * (the DL4MT/Nematus conditional-GRU model) as used by arXiv 1605.04809 as a phrase-based
 * decoder feature function.  sm_100a (B200) only; there is no CPU fallback.
 *
 * Problem statement (§5.1): "We assume ... that the neural model has already
 * been initialized with the source sentence and that the source sentence context is available at
 * all time" (nmt_encode -> context handle); given a set of (hypothesis state, next words), one
 * forward step "(H_i, P_i) <- NMT(H_{i-1}, E_i)" (Alg. 1) yields the word
 * probabilities and the successor states, which are cached at the target nodes and "reused ... as
 * initial states when scoring another batch of hypotheses at later time"
 * (nmt_score_batch -> log-probs + child state handles).  Several models are combined as separately
 * weighted features through the ensemble hook.
 *
 * Conventions (all calls):
 *  - Every call returns nmt_status; NMT_OK = 0.  On error no output array is written and
 *    nmt_last_error() returns a thread-local message naming the offending argument/param/file.
 *  - Pointers marked [host] are host memory, [dev] device memory of the model's device.
 *    The caller owns every input and output array; the library owns models, contexts and
 *    the per-context state arena.  Handles die with nmt_ctx_free.
 *  - Ids are int32 in [0, V); y_prev = -1 denotes BOS (zero embedding).  nmt_state is an opaque
 *    per-context node id (int64).
 *  - A model is immutable after load and may be shared by contexts; calls on one model are
 *    serialised on the model's stream (one writer per context).
 *  - Determinism: identical call sequences give bit-identical outputs on one GPU type.  Child ids
 *    are assigned in first-appearance order of the (parent-major, candidate-order) request stream.
 */
#ifndef NMT_H
#define NMT_H
#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define NMT_API __attribute__((visibility("default")))
#else
#define NMT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NMT_OK = 0,
  NMT_ERR_INVALID_ARG = 1,   /* null pointer, negative count, bad CSR offsets */
  NMT_ERR_IO = 2,            /* params file cannot be opened/read/written */
  NMT_ERR_FORMAT = 3,        /* malformed params header or payload length */
  NMT_ERR_MISSING_PARAM = 4, /* "missing parameter <name>" */
  NMT_ERR_SHAPE = 5,         /* "<name>: expected RxC, got RxC" */
  NMT_ERR_EMPTY_SOURCE = 6,  /* len == 0 */
  NMT_ERR_TOKEN_RANGE = 7,   /* a word id outside [0, V) */
  NMT_ERR_BAD_STATE = 8,     /* unknown / foreign state handle (cf. "unscored expansion") */
  NMT_ERR_CAPACITY = 9,      /* source longer than max_src_len, arena or batch beyond limits */
  NMT_ERR_CUDA = 10,         /* CUDA runtime/driver error, or no sm_100 device */
  NMT_ERR_NCCL = 11,
  NMT_ERR_OOM = 12
} nmt_status;

NMT_API const char* nmt_last_error(void);

typedef enum {
  NMT_PREC_FP32CLASS = 0, /* every GEMM in split bf16x3 (hi*hi + hi*lo + lo*hi), fp32 accumulate;
                             parity bound max|dlogp| <= 1e-3 (BASELINE north_star) */
  NMT_PREC_BF16 = 1       /* single-pass bf16 GEMMs, fp32 accumulate; bound <= 2e-2 */
} nmt_precision;

typedef enum {
  NMT_READOUT_TANH = 0,  /* DL4MT/Nematus deep output: t = tanh(s2 W_l + e W_p + c W_ctx + b) */
  NMT_READOUT_MAXOUT = 1 /* Bahdanau 2014 maxout: t_k = max(pre_2k, pre_2k+1) */
} nmt_readout;

typedef struct {
  int32_t dim_emb;     /* E   (500) */
  int32_t dim_hid;     /* H   (1024); any H <= 1024 (padded to a multiple of 128 on the device) */
  int32_t vocab_src;   /* V_s (50k En / 100k Ru BPE) */
  int32_t vocab_tgt;   /* V_t */
  int32_t max_src_len; /* Tx limit incl. EOS (50 words) */
  nmt_readout readout;
} nmt_dims;

/* Device memory (north_star: "PyTorch is used only for device memory, streams and process groups"):
 * every device allocation of a model - weights, workspaces, state arenas - goes through dev_alloc /
 * dev_free when they are set (e.g. PyTorch's caching allocator: the Python binding passes it), else
 * through a private stream-ordered pool of the model.  Both are called on the calling thread during
 * nmt_* calls, with the model's stream: dev_alloc(bytes, device, stream, alloc_ctx) returns device
 * memory usable in stream order on `stream` (NULL -> NMT_ERR_OOM); dev_free(ptr, bytes, device,
 * stream, alloc_ctx) may reuse it for later work on `stream` at once (work queued before on that
 * stream finishes first).  No allocation after nmt_load synchronises the device.
 * arena_bytes bounds the state arenas (per-context node tables, hash, cached states; live and
 * released contexts): a call that would grow them beyond it first frees released contexts' arenas,
 * then fails with NMT_ERR_CAPACITY before writing any output.  0 = unbounded.                   */
typedef void* (*nmt_dev_alloc_fn)(size_t bytes, int32_t device, void* stream, void* alloc_ctx);
typedef void (*nmt_dev_free_fn)(void* ptr, size_t bytes, int32_t device, void* stream, void* alloc_ctx);

typedef struct {
  int32_t device;          /* CUDA device ordinal */
  nmt_precision precision; /* GEMM recipe, see above */
  int32_t max_src_len;     /* 0 -> 64; at most 65534 and short enough for the attention's shared memory
                              (about 1100 at H = 1024), else NMT_ERR_INVALID_ARG */
  void* stream;            /* cudaStream_t the model's work is issued on; NULL -> a private stream */
  size_t arena_bytes;      /* state-arena budget in bytes, 0 = unbounded (see above) */
  nmt_dev_alloc_fn dev_alloc; /* NULL (with dev_free NULL) -> the model's private pool */
  nmt_dev_free_fn dev_free;
  void* alloc_ctx;         /* passed through to dev_alloc / dev_free */
} nmt_opts;

typedef struct nmt_model nmt_model;
typedef struct nmt_ctx nmt_ctx;
typedef struct nmt_ensemble nmt_ensemble;
typedef int64_t nmt_state;

/* ---- models -------------------------------------------------------------------------------
 * Params container ("text header + little-endian float32 payload"):
 *   "NMTPARAMS 1\n" "dims E H Vs Vt readout=<tanh|maxout> eos=<id> unk=<id>\n" "arrays n\n"
 *   n lines "<name> <rows> <cols>\n" (Nematus names), zero padding to 64 bytes,
 *   then the arrays row-major float32 LE in header order.  Every required name must be present
 *   (NMT_ERR_MISSING_PARAM), shapes must agree with dims (NMT_ERR_SHAPE), the payload length must
 *   be exact (NMT_ERR_FORMAT).  Weights are re-laid out on the device at load (bf16 K-major
 *   tiles, hi/lo splits, precomputed embedding projections); the model also keeps the container
 *   bytes on the host so that nmt_save_params can write them back unchanged.                   */
NMT_API nmt_status nmt_load(const char* params_path, const nmt_opts* opts, nmt_model** out);
NMT_API nmt_status nmt_load_buffer(const void* buf /*[host]*/, size_t len, const nmt_opts* opts, nmt_model** out);
NMT_API nmt_status nmt_model_dims(const nmt_model* m, nmt_dims* out);
/* Device bytes the model holds through its allocator now (live) and at most so far (peak), and the
 * state-arena bytes counted against nmt_opts.arena_bytes (arena); any pointer may be NULL.       */
NMT_API nmt_status nmt_model_memory(const nmt_model* m, size_t* live, size_t* peak, size_t* arena);
/* Checkpoint averaging (NMT-k-Avg: "the element-wise average of all model weights in
 * the NMT ensembles", saved as a new model).  bufs[n] / lens[n] [host] are n params containers with
 * IDENTICAL headers (dims, readout, array names and shapes; else NMT_ERR_SHAPE naming the first
 * difference, NMT_ERR_FORMAT for a malformed container); out [host] receives a container of the
 * same layout (out_len must equal lens[0], else NMT_ERR_INVALID_ARG) whose payload is, per element,
 * fp32(sum_i x_i / n) with the sum taken in fp64 in member order on `device`.  Load it with
 * nmt_load_buffer.  Synchronous; the caller owns every buffer.                                   */
NMT_API nmt_status nmt_params_average(int32_t n, const void* const* bufs, const size_t* lens, int32_t device,
                                      void* out, size_t out_len);
/* Writes the model's params container to `path`, byte-identical to the container it was loaded or
 * generated from (SPEC.md:192 round trip).  NMT_ERR_IO if the file cannot be written.           */
NMT_API nmt_status nmt_save_params(const nmt_model* m, const char* path);
/* The same bytes into out [host]: out == NULL -> *len = size needed; *len < size ->
 * NMT_ERR_CAPACITY (and *len = size).                                                           */
NMT_API nmt_status nmt_params_bytes(const nmt_model* m, void* out, size_t* len);
/* Seeded synthetic model (SURVEY §8(d) generator): embeddings N(0,1), linear maps
 * N(0, 1/fan_in), orthogonal recurrent blocks (Haar, DL4MT ortho_weight), biases N(0, 0.1^2),
 * U_att N(0, (2/sqrt(2H))^2), W_o scaled so that std(t.W_o) ~ logit_std, b_o[w] = -ln(w+1).
 * Counter-based draws (splitmix64 + Box-Muller, keyed by seed and array name): the same
 * (dims, seed, logit_std) always gives the same bytes; it does NOT reproduce synth/'s numpy
 * stream.  nmt_random_params is host-only (no GPU needed): out == NULL -> *len = size; otherwise
 * writes the container (NMT_ERR_CAPACITY if *len is too small).  nmt_create_random = generate +
 * nmt_load_buffer (dims->max_src_len is used when opts->max_src_len == 0).  Bad dims or
 * logit_std <= 0 -> NMT_ERR_INVALID_ARG.                                                         */
NMT_API nmt_status nmt_random_params(const nmt_dims* d, uint64_t seed, float logit_std, void* out, size_t* len);
NMT_API nmt_status nmt_create_random(const nmt_dims* d, uint64_t seed, float logit_std, const nmt_opts* opts,
                                     nmt_model** out);
/* Releases the caller's handle; the device memory goes when the last context of the model is freed
 * too (models and contexts may be freed in any order). */
NMT_API void nmt_model_free(nmt_model* m);

/* ---- source context --------------------------------------------------------
 * Bidirectional-GRU encoder over src_ids[0..len) [host] (the caller appends EOS, Nematus
 * convention); computes ctx = [fwd_j ; bwd_j], s_0 = tanh(mean_j ctx_j W_init + b_init) and the
 * attention keys pctx = ctx Wc_att + b_att.  len == 0 -> NMT_ERR_EMPTY_SOURCE; len > max_src_len
 * -> NMT_ERR_CAPACITY.  The returned context owns a state arena whose root node is (s_0, BOS).  */
NMT_API nmt_status nmt_encode(nmt_model* m, const int32_t* src_ids, int32_t len, nmt_ctx** out);
NMT_API nmt_state nmt_root(const nmt_ctx* c);
/* Same with src_ids [dev] (e.g. resident in HBM); token ids are validated on the device and an
 * out-of-range id is reported by nmt_ctx_check().  Asynchronous on the model stream.            */
NMT_API nmt_status nmt_encode_dev(nmt_model* m, const int32_t* src_ids, int32_t len, nmt_ctx** out);
/* n sources at once (one context per sentence): ids [host] holds the
 * sentences back to back, offsets [host, n+1] (offsets[0] = 0, non-decreasing) delimits them, and
 * outs[n] [host] receives one context per sentence in input order.  The recurrences of all
 * sentences advance together, one tensor-core GEMM per time step over the sentences still running
 * (tensor-bound when hundreds of sentences are batched); results agree with
 * nmt_encode within the precision's tolerance, not bit for bit.  Errors as nmt_encode, checked for
 * every sentence before any work (the message names the sentence); on error no context is created.
 * n == 0 is a no-op.  Up to 8 sentences are encoded one by one with nmt_encode's kernel (faster
 * there).  Asynchronous on the model stream.                                                    */
NMT_API nmt_status nmt_encode_batch(nmt_model* m, int32_t n, const int32_t* ids, const int32_t* offsets,
                                    nmt_ctx** outs);
/* Releases the context; its arena is kept by the model for reuse by a later nmt_encode. */
NMT_API void nmt_ctx_free(nmt_ctx* c);

/* ---- batched scoring (Alg. 1; parent-indexed rows, DESIGN.md §2 A13) -----
 * parents[n_parents], cand_offsets[n_parents+1] (CSR, offsets[0] = 0, non-decreasing) and
 * cand_words[N_cand] are [host].  For every candidate i of parent k:
 *   out_logprob[i] = log p(cand_words[i] | parent k)  (log-softmax over the WHOLE target vocab,
 *                    PAPER.md:107; the logits are never materialised)
 *   out_child[i]   = state handle of the node (parent k, word) - interned: the same (parent,
 *                    word) pair always yields the same handle and a bit-identical log-prob.
 * out_argmax[n_parents] (may be NULL) = most probable next word of each parent (lowest id on
 * ties), -1 for a parent with no candidates.  Each distinct parent with >= 1 candidate that was
 * never stepped is stepped once (GRU1 -> attention -> GRU2 -> readout -> vocab log-softmax) and
 * its (s2, t, logZ, argmax) cached; later calls reuse it.  N_cand == 0 is a no-op.           */
NMT_API nmt_status nmt_score_batch(nmt_ctx* c, int32_t n_parents, const nmt_state* parents,
                           const int32_t* cand_offsets, const int32_t* cand_words,
                           float* out_logprob, nmt_state* out_child, int32_t* out_argmax);

/* Same, device-resident: all pointers [dev]; int32 parents/children (node ids < 2^31);
 * n_cand must equal cand_offsets[n_parents].  Issued asynchronously on the model stream, no host
 * synchronisation; invalid ids are reported by the next nmt_ctx_check().                     */
NMT_API nmt_status nmt_score_batch_dev(nmt_ctx* c, int32_t n_parents, const int32_t* parents,
                               const int32_t* cand_offsets, int32_t n_cand, const int32_t* cand_words,
                               float* out_logprob, int32_t* out_child, int32_t* out_argmax);
/* Several sentences in one call: parent k is a state of ctx_per_parent[k] [host,
 * n_parents; all contexts of one model, else NMT_ERR_INVALID_ARG]; every other argument, output
 * and error as nmt_score_batch, in input order (child handles belong to their parent's context).
 * All contexts' new rows go through ONE fused decoder step (each row attends over its own
 * sentence and writes its own arena; every context's rows start at a multiple of 4), with one
 * planner pass and one gather-dot over all contexts and one host synchronisation.  Child ids are
 * those per-context nmt_score_batch calls would give; log-probs agree with them up to fp32
 * summation order (split-K factors depend on the fused row count).                             */
NMT_API nmt_status nmt_score_batch_multi(int32_t n_parents, nmt_ctx* const* ctx_per_parent, const nmt_state* parents,
                                         const int32_t* cand_offsets, const int32_t* cand_words, float* out_logprob,
                                         nmt_state* out_child, int32_t* out_argmax);
/* ---- beam step (pure-NMT beam search on the same step) ----
 * For each parent (steps it first if it was never stepped), the k highest log-prob next words over
 * the WHOLE target vocabulary.  parents [host] n_parents state handles; out_words [host] int32,
 * out_logprob [host] float and out_child [host] state handles, each [n_parents * k], row-major by
 * parent, descending log-prob (ties: lower word id).  The k words are chosen from the vocabulary
 * GEMM's logits (a top-k epilogue, no logits in HBM), in the model's precision; their log-probs and
 * child states are exactly those nmt_score_batch returns for the same (parent, word).
 * 1 <= k <= NMT_TOPK_MAX (else NMT_ERR_INVALID_ARG); unknown parent -> NMT_ERR_BAD_STATE.        */
#define NMT_TOPK_MAX 8
NMT_API nmt_status nmt_beam_step(nmt_ctx* c, int32_t n_parents, const nmt_state* parents, int32_t k,
                                 int32_t* out_words, float* out_logprob, nmt_state* out_child);
/* ScoreBatch (Alg. 1) in one call.  Pair i expands hypothesis state hyp_states[i]
 * [host] by the phrase phrase_words[phrase_offsets[i] .. phrase_offsets[i+1]) [host] (1..16 words;
 * an empty phrase -> NMT_ERR_INVALID_ARG "empty expansion").  The library builds the
 * forest of per-hypothesis prefix trees, runs ONE batched step per tree depth
 * (shared prefixes collapse, states are cached for later calls) and
 * returns out_logp[i] = sum of the phrase's word log-probs and out_state[i] = the state after the
 * phrase [host, n_pairs each].  stats [host, 33 int32, may be NULL]: [0] = steps (= the longest
 * phrase), [1..16] = collapsed edges (word-scores) per depth, [17..32] = decoder
 * rows stepped per depth.                                                                        */
NMT_API nmt_status nmt_score_forest(nmt_ctx* c, int32_t n_pairs, const nmt_state* hyp_states,
                                    const int32_t* phrase_offsets, const int32_t* phrase_words, float* out_logp,
                                    nmt_state* out_state, int32_t* stats);
/* ScoreBatch over several sentences at once: pair i expands hyp_states[i], a state of
 * ctx_per_pair[i] [host, n_pairs; contexts of one model], by its phrase (as nmt_score_forest, any
 * length).  Each depth is ONE fused multi-context step (nmt_score_batch_multi), so the stacks of
 * many sentences share the decoder GEMMs; shared prefixes collapse per context.  out_logp [host]
 * = the phrase's summed log-prob, out_state [host] = the state after it (a state of that pair's
 * context).  Errors as nmt_score_batch_multi; outputs are written only on success.             */
NMT_API nmt_status nmt_score_forest_multi(int32_t n_pairs, nmt_ctx* const* ctx_per_pair, const nmt_state* hyp_states,
                                          const int32_t* phrase_offsets, const int32_t* phrase_words,
                                          float* out_logp, nmt_state* out_state);
/* n-best forced rescoring (rescoring gives "the same as if they
 * were produced at decode-time"): sequence i = words[offsets[i] .. offsets[i+1]) [host] (non-empty,
 * any length; the caller appends EOS) is scored from the root: out_logp[i] = sum_j log p(w_j | w_<j)
 * and out_state[i] = the state after it [host, n each].  All sequences form one prefix forest, so
 * shared prefixes are stepped once and each depth is one batched step (as nmt_score_forest).    */
NMT_API nmt_status nmt_score_sequences(nmt_ctx* c, int32_t n, const int32_t* offsets, const int32_t* words,
                                       float* out_logp, nmt_state* out_state);
/* Waits for the model stream and reports a device-side validation error of earlier _dev calls. */
NMT_API nmt_status nmt_ctx_check(nmt_ctx* c);
/* Grows the context's arena to hold n_nodes nodes and n_stepped stepped nodes without further
 * reallocation (a decoder that knows its stack sizes avoids the doubling copies).  Never shrinks. */
NMT_API nmt_status nmt_ctx_reserve(nmt_ctx* c, int64_t n_nodes, int64_t n_stepped);
/* Number of nodes and stepped nodes in the context's arena (synchronises the stream). */
NMT_API nmt_status nmt_ctx_stats(nmt_ctx* c, int64_t* n_nodes, int64_t* n_stepped);

/* ---- synthetic parents (bench / tests): n nodes with given input state s[n x H] [host] and
 * previous word y_prev[n] [host] (-1 = BOS), not children of any node.  Pageable arrays are
 * copied before the call returns; page-locked arrays are read asynchronously (the upload overlaps
 * the encoder) and must stay unchanged until the next synchronising call on the context
 * (nmt_score_batch, nmt_score_forest, nmt_beam_step, nmt_ctx_check, nmt_ctx_stats) returns.      */
NMT_API nmt_status nmt_inject_states(nmt_ctx* c, int32_t n, const float* s, const int32_t* y_prev, nmt_state* out);

/* Device variant: s [dev, n x H floats], y_prev [dev, n], out [dev, n int32 node ids]; async.  */
NMT_API nmt_status nmt_inject_states_dev(nmt_ctx* c, int32_t n, const float* s, const int32_t* y_prev, int32_t* out);

/* ---- diagnostics (bench.py) -----------------------------------------------------------------
 * nmt_launch_count: kernels this library has launched in the process so far.
 * nmt_profile: 0 off, 1 CUDA events around the vocabulary GEMM only, 2 around every stage (on the
 * model stream).  nmt_profile_read synchronises and returns the milliseconds and launch counts per
 * stage accumulated since the previous read, stage order:
 *   0 plan  1 gather  2 gemm_h1  3 gru1  4 gemm_q  5 attention  6 gemm_g2  7 gru2  8 gemm_ro
 *   9 readout  10 vocab_gemm_lse  11 finalize  12 gather_dot  13 enc_gather  14 enc_gemm_in
 *   15 enc_recurrence  16 enc_init  17 enc_pctx  18 inject                                        */
#define NMT_N_STAGES 19
NMT_API long long nmt_launch_count(void);
NMT_API nmt_status nmt_profile(nmt_model* m, int32_t mode);
NMT_API nmt_status nmt_profile_read(nmt_model* m, double* ms, int64_t* count);

/* ---- test-only exports ----------------------------------------------------------------------- */
/* live device allocations of every model of the process (count, bytes): 0 after all are freed     */
NMT_API nmt_status nmt_device_allocations(int64_t* count, size_t* bytes);
/* models and contexts (live or pooled) that exist in the process                                 */
NMT_API nmt_status nmt_debug_live_objects(int64_t* models, int64_t* contexts);
/* full log-prob row of one node over the whole vocab (normalisation tests); steps the node if
 * needed.  out [host, vocab_tgt floats]                                                          */
NMT_API nmt_status nmt_logprobs_full(nmt_ctx* c, nmt_state node, float* out);
/* encoder outputs: ctx [Tx x 2H], pctx [Tx x 2H], s0 [H]; any pointer may be NULL [host]         */
NMT_API nmt_status nmt_debug_encoder(nmt_ctx* c, float* ctx, float* pctx, float* s0);
/* per-stage intermediates of one node's step (without caching): s1[H], alpha[Tx], c[2H], s2[H],
 * t[E], logZ[1], argmax[1]; any pointer may be NULL [host].  The step forms c explicitly (D5); the
 * scoring calls of a single context fold it into D6/D7 as alpha . (ctx . W) (reading A31),
 * equal up to the precision's operand rounding.                                                   */
NMT_API nmt_status nmt_debug_intermediates(nmt_ctx* c, nmt_state node, float* s1, float* alpha, float* ctxv,
                                   float* s2, float* t, float* logZ, int32_t* argmax);
/* The vocabulary stage alone (D8 + D9, SURVEY §8(b) "minimum slice"): R rows of readout outputs
 * t [host, R x dim_emb] -> out_logZ [host, R] = logsumexp_v(t.W_o + b_o), out_argmax [host, R or
 * NULL] (lowest id on ties) and, for the CSR candidates cand_offsets [R+1] / cand_words [N_cand],
 * out_logprob [host, N_cand] = t.W_o[:,w] + b_o[w] - logZ.  Same kernels as a step (vocabulary
 * GEMM with the fused log-sum-exp, finalize, gather-dot), run on a scratch context.             */
NMT_API nmt_status nmt_debug_vocab(nmt_model* m, int32_t R, const float* t, const int32_t* cand_offsets,
                                   const int32_t* cand_words, float* out_logprob, float* out_logZ,
                                   int32_t* out_argmax);
/* The vocab-parallel path of one step (nmt_vocab_shard) emulated on one GPU: the vocabulary is cut
 * into n_slices 256-column-aligned slices computed one after the other, as ranks 0..n-1 would,
 * and their per-row (max, sum exp, argmax) partials are merged by the same combine kernel that runs
 * after the all-gather.  t, out_logZ, out_argmax as nmt_debug_vocab.                          */
NMT_API nmt_status nmt_debug_vocab_shards(nmt_model* m, int32_t R, const float* t, int32_t n_slices, float* out_logZ,
                                          int32_t* out_argmax);
/* GEMM engine unit test: C[M x N] = A[M x K] . B[K x N] (+ bias[N]) with the tcgen05 kernel;
 * split = 1 -> bf16x3.  A, B, bias, C are [host] fp32 row-major; N % 128 == 0, K % 64 == 0.     */
NMT_API nmt_status nmt_test_gemm(int32_t M, int32_t N, int32_t K, int32_t split, const float* A, const float* B,
                         const float* bias, float* C);

/* GEMM engine micro-benchmark on device-resident random operands: average ms of `iters` launches
 * of C[M x N] = A[M x K].B[K x N] (epi 0: fp32 store, N % 128 == 0; epi 1: vocabulary online
 * log-sum-exp, N % 256 == 0), split = bf16x3, ksplit = split-K factor (epi 0).                 */
NMT_API nmt_status nmt_bench_gemm(int32_t M, int32_t N, int32_t K, int32_t split, int32_t epi, int32_t ksplit,
                                  int32_t iters, float* ms_out);

/* ---- vocab-parallel scoring (PAPER.md:98 multi-GPU) ---------------------
 * Every rank (one per GPU) holds the same model and issues the same calls; after this call the
 * rank's vocabulary GEMM covers only its slice of the target vocabulary (the 256-column tiles
 * [T*rank/world, T*(rank+1)/world)), each row's (max, sum exp, argmax) over the slice is exchanged
 * with ONE all-gather per step on `comm` (an nmt_ensemble communicator of `world` ranks: 16 B per
 * row per rank) and merged in rank order, so logZ, argmax and every log-prob equal the single-GPU
 * result up to fp32 summation order.  The rest of the step is replicated.  world == 1 or
 * comm == NULL restores the full vocabulary.  rank/world must match the communicator.             */
NMT_API nmt_status nmt_vocab_shard(nmt_model* m, int32_t rank, int32_t world, nmt_ensemble* comm);

/* ---- ensemble hook and communicators (models as separately weighted features;
 * north_star: members on separate GPUs, per-word probabilities combined over NVLink) ------------
 * A communicator (nmt_ensemble) joins n members (or vocab-parallel ranks, nmt_vocab_shard) and has
 * one of two transports:
 *  - NCCL (nmt_ensemble_init): one member per process/GPU.  nccl_unique_id points to the 128-byte
 *    ncclUniqueId made by rank 0 with nmt_ensemble_get_unique_id and broadcast by the harness (torch
 *    process group).  NCCL is loaded at run time (NMT_ERR_NCCL if it cannot be).
 *  - local (nmt_ensemble_init_local): all n members in THIS process, each driven by its own host
 *    thread; devices[n] [host] (NULL -> all on device 0) may repeat, so several members can share a
 *    GPU.  out[n] [host] receives one handle per rank; free each.  A collective waits up to 120 s for
 *    every member's thread (then NMT_ERR_INVALID_ARG).
 * nmt_ensemble_combine: member `rank` contributes member_logprob [dev, n floats, on its model's
 * device] with its weight; every member's row is all-gathered, and the root writes out [dev, n]
 * (ignored elsewhere) combining the members IN MEMBER ORDER (fp64 accumulation, deterministic):
 *    mode 0 (log-linear):   out = sum_m w_m logp_m
 *    mode 1 (interpolate):  out = mx + log sum_m w_m exp(logp_m - mx),  mx = max_m logp_m  (w_m >= 0)
 * Issued asynchronously on `stream` (the member's model stream, or any stream ordered after the
 * producer of member_logprob).  Every member must call it with the same n, mode and root.       */
NMT_API nmt_status nmt_ensemble_init(int32_t n_members, int32_t rank, const void* nccl_unique_id, int32_t device,
                             nmt_ensemble** out);
NMT_API nmt_status nmt_ensemble_init_local(int32_t n_members, const int32_t* devices, nmt_ensemble** out);
NMT_API nmt_status nmt_ensemble_get_unique_id(void* out128);
NMT_API nmt_status nmt_ensemble_combine(nmt_ensemble* e, const float* member_logprob, int32_t n, float weight,
                                int32_t mode, int32_t root, float* out, void* stream);
NMT_API void nmt_ensemble_free(nmt_ensemble* e);

#ifdef __cplusplus
}
#endif
#endif /* NMT_H */
