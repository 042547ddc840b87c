// kernels.h - device-side views and launchers of the non-GEMM kernels (kernels.cu).
#pragma once
#include "internal.h"

namespace nmt {

// CNT_BIGP: set (atomicOr) by the pctx producers when some |2 pctx| > kAttnExpClamp, i.e. exp(2 pctx) was
// clamped; the attention then takes its tanh path for the context (reset with the context)
enum { CNT_NODES = 0, CNT_SLOTS = 1, CNT_ERR = 2, CNT_R = 3, CNT_BIGP = 4, CNT_N = 5 };
// exp(+-21): a pair product (1 + e^2p e^2q)(1 + e^2p' e^2q') <= e^84.x stays inside the normal fp32 range and
// below the reciprocal seed's limit (bits < 0x7EF311C3); |p|, |q| > 10.5 take the tanh path
constexpr float kAttnExpClamp = 21.f;
enum { ERR_BAD_STATE = 1, ERR_TOKEN = 2, ERR_OFFSETS = 4 };

// Per-context device arena + node table + (parent, word) -> child hash (the state cache).
struct CtxDev {
  int* counters;               // [CNT_N]
  int* node_word;              // y_prev of each node's step (-1 BOS)
  int* node_parent;            // -1 for the root / injected nodes
  int* node_src;               // input slot of parentless nodes
  int* node_slot;              // stepped output slot, -1 if not stepped
  int* node_claim;             // scratch for deterministic parent dedup (INT_MAX when idle)
  unsigned long long* hkeys;   // (parent << 32 | word), -1 empty
  int* hvals;                  // child id (>= 0), or claim (< 0) during a call
  uint64_t hmask;
  float* S;                    // [slots][Hp] states (slot 0 = s0, slot 1 = scratch)
  float* T;                    // [slots][Ep] readout outputs t
  float* logZ;                 // [slots]
  int* amax;                   // [slots]
  int V, H, Hp, Ep;
};

// One call's request (device pointers) and planner scratch.
struct PlanIO {
  int n_par, n_cand;
  const int* parents;   // [n_par]
  const int* offsets;   // [n_par + 1]
  const int* words;     // [n_cand]
  int* cand_k;          // [n_cand] parent index of each candidate
  int* cand_hslot;      // [n_cand] hash slot (-1 invalid)
  int* row_src;         // [n_par] input slot of each stepped row
  int* row_y;           // [n_par] previous word of each row
  int* row_dst;         // [n_par] output slot of each row
  int* row_node;        // [n_par] node id of each row
  int* cflag;           // [n_cand] first appearance of a new key
  int* pflag;           // [n_par] parent must be stepped
  int* bcount;          // [blocks] per-block flag counts
  int* snap;            // [2] node / slot counters at plan start
  int step_all;         // 1: step every listed parent not yet stepped, candidates or not (beam step)
};

// One context of a multi-context step (nmt_score_batch_multi): its arena and attention source.
struct GrpStep {
  float* S;
  float* T;
  float* logZ;
  int* amax;
  const float* pctx;
  const float* ctx;
  int Tx;
  const float* epctx;  // exp(2 pctx) (clamped) [Tx][Cp]
  const int* counters;  // the context's counters (CNT_BIGP)
};

// Planner / gather-dot descriptor of one context of a multi-context call (blockIdx.y = group).
struct PlanDesc {
  CtxDev c;
  PlanIO io;          // request and planner scratch slices of this group
  int* R_out;         // the group's stepped-row count
  float* out_logp;    // outputs of this group's candidates / parents
  int* out_child;
  int* out_argmax;
};

// Decoder-step workspace view (rows r < *R).
struct StepDev {
  const int* row_grp;  // multi-context step: group of each row (else null); rows with row_dst < 0 are dead
  const GrpStep* gs;   // multi-context step: per-group arenas (else null)
  const int* R;
  const int* row_src;
  const int* row_y;
  const int* row_dst;
  int V, H, Hp, Cp, E, Ep, ROp, maxout;
  __nv_bfloat16* A_s; int lda_s, lo_s;   // [R][sf*Hp]
  float* G1;                             // [ks_g1][R..][3Hp] split-K partials (stride ps_g1 floats)
  const float* Ex;                       // [V+1][3Hp]
  float* S1;                             // [R][Hp]
  __nv_bfloat16* X; int ldx, lo_x;       // [R][sf*(Hp+Cp+Hp)]  [s1 | c | s2]
  float* Q;                              // [ks_q][R..][Cp]
  float* Cf;                             // [R][Cp]
  float* alpha_out; int alpha_ld;        // [R][max_src_len] (may be null)
  float* G2;                             // [..][R..][4Hp]: ks_g2[0] | [1] | [2] partials of gates | hUx | cWcx
  const float* b_nl;                     // [2Hp]
  const float* bx_nl;                    // [Hp]
  float* RO;                             // [ks_ro][R..][ROp]
  const float* Eproj;                    // [V+1][ROp]
  __nv_bfloat16* A_t; int lda_t, lo_t;   // [R][sf*Ep]
  float4* part; int n_tiles;             // [R][2 * cpm] LSE partials of the vocabulary GEMM
  const int* cpm;                        // runs per m-tile (device, written by the GEMM)
  float4* xout;                          // vocab-parallel: finalize writes each row's (max, sum exp,
                                         // argmax) of this rank's vocabulary slice here (else null)
  int ks_g1, ks_q, ks_g2[3], ks_ro;      // split-K partial counts of the decoder GEMM outputs
  int64_t ps_g1, ps_q, ps_g2, ps_ro;     // floats between consecutive partials
  int diag_attn_slow;                    // (diagnostic builds: force the attention's tanh path)
  int proj_k;                            // projected-context step: attention writes alpha (bf16 hi | lo,
                                         // zero past Tx) to X columns [Hp, Hp + proj_k) instead of c; 0: c
};

struct AttnCtx {
  const float* pctx;   // [Tx][Cp]
  const float* ctx;    // [Tx][Cp]
  const float* U_att;  // [Cp]
  float c_tt;
  int Tx;
  const float* epctx;   // [Tx][Cp] exp(2 pctx), exponent clamped to +-kAttnExpClamp
  const int* counters;  // the context's counters (CNT_BIGP: some exponent was clamped)
};

struct EncDev {
  int H, Hp, NB, UPC, Vs;
  unsigned epoch;        // 1..65535, per encode: target of the tail grid barrier's growing counter
  long long* trace;      // diagnostic (NMT_ENC_TRACE): [Tx][8] clock64 phase stamps of CTA 0, thread 0
  const float* Uarr;     // [2][NB][3*UPC][Hp] recurrent weights per CTA (rows zero-padded to Hp)
  const int* src;        // [Tx] source ids (device)
  const float* encin;    // [Vs][6Hp] precomputed x.[W|Wx] + [b|bx] of both directions per source word
  float* ctx;            // [Tx][2Hp]
  __nv_bfloat16* ctxbf;  // [Tx][4Hp] hi | lo copy for the pctx GEMM
  unsigned* hx;          // [2 dirs][2 parities][Hp] fp32 h with the tag (t + 1) mod 4 in the 2 low bits (zero between encodes)
  float* mean;           // [2H] mean_j ctx_j (real indices)
  int* bar;              // [1] tail grid barrier
  int* err;              // validation flags of the context
  const float* W_initT;  // [H][2H] ff_state_W transposed (contiguous per output)
  const float* b_init;   // [H]
  float* S0;             // [H] arena slot 0
};

// nmt_encode_batch: n sentences sorted by length (descending); token rows sentence-major
struct EncBatchDev {
  int n, H, Hp;
  const int* src;        // [n_tok] source ids
  const int* tok_off;    // [n + 1] first token row of each sentence
  const int* row_b;      // [n_tok] sentence of each token row
  const float* encin;    // [Vs][6Hp] precomputed input projections (EncDev::encin)
  const float* G; int ks; int64_t ps;  // [n][6Hp] recurrent GEMM output (+ split-K partials)
  float* h;              // [n][2Hp] fp32 states [fwd | bwd]
  __nv_bfloat16* A; int lo_a;  // [n][4Hp] bf16 operand of the next step's GEMM (hi | lo at +2Hp)
  __nv_bfloat16* ctxbf;  // [n_tok][4Hp] hi | lo copy of ctx (pctx GEMM operand)
  __nv_bfloat16* Am;     // [n][4Hp] mean ctx hi | lo (s0 GEMM operand)
  float* const* ctx;     // [n] per-sentence ctx [Tx][Cp]
  float* const* pctx;    // [n] per-sentence pctx [Tx][Cp]
  float* const* epctx;   // [n] per-sentence exp(2 pctx) [Tx][Cp] (clamped)
  int* const* cnt;       // [n] per-sentence counters (CNT_BIGP)
  float* const* S0;      // [n] slot 0 of each sentence's state arena
  const float* b_init;   // [H]
  const float* b_att;    // [Cp]
};

enum { EW_GATHER, EW_GRU1, EW_ATTN, EW_GRU2, EW_READOUT, EW_FINALIZE };

void pack_T(const float* src, int ld_src, int K, int N, __nv_bfloat16* dst, int ld_dst, int row0, int col0, int rmap,
            int kmap, int H, int Hp, int lo_off, cudaStream_t st);
void pack_rows(const float* src, int ld_src, int rows, int K, __nv_bfloat16* dst, int ld_dst, int col0, int lo_off,
               cudaStream_t st);
void to_panels(const __nv_bfloat16* src, int rows, int cols, __nv_bfloat16* dst, cudaStream_t st);
void transpose_f32(const float* src, int K, int N, float* dst, int ld_dst, cudaStream_t st);
void avg_accum(double* acc, const float* x, int64_t n, bool first, cudaStream_t st);
void avg_finish(float* out, const double* acc, int64_t n, int members, cudaStream_t st);
void beam_gather(const StepDev& d, const CtxDev& c, const int* parents, int n, cudaStream_t st);
void topk_merge(const float2* topk, const int* cpm_dev, int n, int k, int* out_words, cudaStream_t st);
void ctx_reset(const CtxDev& c, int64_t hcap, cudaStream_t st);
void fill_i32(int* p, int64_t n, int v, cudaStream_t st);
void plan(const CtxDev& c, const PlanIO& io, int* R_dev, cudaStream_t st);
// G groups at once: descs [dev, G]; max_cand / max_par = the largest group's counts
void plan_multi(const PlanDesc* descs, int G, int max_cand, int max_par, cudaStream_t st);
void rehash(const unsigned long long* okeys, const int* ovals, int64_t ocap, unsigned long long* nkeys, int* nvals,
            uint64_t nmask, cudaStream_t st);
void inject(const CtxDev& c, int n, const float* s, const int* y, int* out_ids, int* done, cudaStream_t st);
void step_elementwise(int which, const StepDev& d, const AttnCtx& a, float* S, float* T, float* logZ, int* amax,
                      int R_max, cudaStream_t st);
void gather_dot(const CtxDev& c, const PlanIO& io, const float* Wo32, const float* bo, int Ep, float* out_logp,
                int* out_child32, long long* out_child64, int* out_argmax, cudaStream_t st);
// the CNT_N counters of every group's context into out [dev, G x CNT_N] (one D2H for the call)
// vocab-parallel combine: xall [world][stride] (max, sum exp, argmax) of each rank's slice, merged in
// rank order (ties -> the lower rank's = lower word id) -> logZ, argmax of every row into the arena
void shard_combine(const StepDev& d, const float4* xall, int world, int stride, float* logZ, int* amax, int R_max,
                   cudaStream_t st);
void counters_multi(const PlanDesc* descs, int G, int* out, cudaStream_t st);
void gather_dot_multi(const PlanDesc* descs, int G, int max_cand, int max_par, const float* Wo32, const float* bo,
                      int Ep, cudaStream_t st);
void gather_idx(const int* src, const int* idx, int n, int* out, cudaStream_t st);
void path_sum(const float* logp, const int* child, const int* off, const int* pos, int n, float* out_logp,
              int* out_state, cudaStream_t st);
void full_row(const float* T, const float* Wo32, const float* bo, const float* logZ, int slot, int Ep, int V,
              float* out, cudaStream_t st);
void enc_recur(const EncDev& e, int Tx, cudaStream_t st);
// dynamic shared memory of the attention kernel for Cp context columns, Tx source positions and
// `rpb` rows per CTA (load-time check of max_src_len against the 227 KB per-CTA limit)
size_t attention_smem_bytes(int Cp, int Tx, int rpb);
void encb_gates(const EncBatchDev& e, int t, int active, cudaStream_t st);
void encb_mean(const EncBatchDev& e, cudaStream_t st);
void encb_s0(const EncBatchDev& e, const float* S0w, int ks, int64_t ps, cudaStream_t st);
void encb_pctx(const EncBatchDev& e, const float* P, int ks, int64_t ps, int n_tok, cudaStream_t st);
void ctx_reset_many(const CtxDev* cs, const int64_t* hcaps, int n, int64_t hcap_max, cudaStream_t st);

}  // namespace nmt
