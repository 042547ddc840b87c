// internal.h - shared declarations of the libnmt host runtime and kernel launchers.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>

#include "../../include/nmt.h"

namespace nmt {

constexpr int kNumSMs = 148;  // B200

struct NmtError {
  nmt_status code;
  std::string msg;
  NmtError(nmt_status c, std::string m) : code(c), msg(std::move(m)) {}
};

#define CK(expr)                                                                                           \
  do {                                                                                                     \
    cudaError_t _e = (expr);                                                                               \
    if (_e != cudaSuccess)                                                                                 \
      throw ::nmt::NmtError(_e == cudaErrorMemoryAllocation ? NMT_ERR_OOM : NMT_ERR_CUDA,                   \
                            std::string(#expr) + ": " + cudaGetErrorString(_e));                          \
  } while (0)

// every kernel launch of the library goes through CK_LAUNCH (counted for the bench's gpu_launches)
void note_launch();
#define CK_LAUNCH()            \
  do {                         \
    ::nmt::note_launch();      \
    CK(cudaGetLastError());    \
  } while (0)

// The > 48 KB dynamic shared-memory opt-in is a per-device-context attribute of a kernel: set it once per
// (kernel, device) at the largest size requested so far (thread-safe; models may live on several devices
// and be driven by several threads).  `per_dev` is a function-local static of the launch site.
constexpr int kMaxDevices = 64;
extern std::mutex g_attr_mu;
template <typename K>
inline void ensure_smem_attr(K* kernel, std::atomic<size_t>* per_dev, size_t smem) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) throw NmtError(NMT_ERR_CUDA, "device ordinal beyond kMaxDevices");
  if (smem <= per_dev[dev].load(std::memory_order_acquire)) return;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if (smem <= per_dev[dev].load(std::memory_order_relaxed)) return;
  CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  per_dev[dev].store(smem, std::memory_order_release);
}

// Launch with the programmatic-stream-serialization attribute (PDL): the kernel may start while the
// previous kernel of the stream drains; every kernel calls pdl_wait() before touching its inputs.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

// --------------------------------------------------------------------------- GEMM engine
struct GemmShape {
  int M;             // rows (if M_dev == nullptr)
  const int* M_dev;  // device-resident row count (dynamic batch size), or nullptr
  int N;             // output columns, multiple of the N tile
  int a_col0;        // first column of A used
  int a_lo_off;      // split: column offset of A's lo half relative to the hi column
  int b_lo_off;      // split: column offset of B's lo half
  int passes;        // 1 (bf16) or 3 (bf16x3: hi.hi + hi.lo + lo.hi)
  int nreg;          // number of N regions (>= 1)
  int reg_n_end[4];  // region r covers output columns [reg_n_end[r-1], reg_n_end[r])
  int reg_k0[4];     // K range [k0, k1) of region r (multiples of 64, relative to a_col0 / 0)
  int reg_k1[4];
  int ksplit;        // split-K factor: split s writes its partial sum to out + s * split_stride
  int reg_ks[4];     // per-region split-K factor (0: ksplit); regions may split differently so that
                     // every work item carries about the same number of k-blocks
  int b_panel_rows;  // 0: B is [N][K] row-major; else B is stored as k-block panels [K/64][b_panel_rows][64]
                     // (every TMA box is one contiguous chunk): coordinate (0, kb * b_panel_rows + row)
  int n_off;         // EPI_LSE / EPI_TOPK: first B row (= vocabulary column) of the GEMM's N range (vocab
                     // slice of a vocab-parallel rank); reported columns are global
  // second B operand (EPI_GRU2 / EPI_READOUT, the tensor map in the tmC slot): k-blocks [b2_kb0, b2_kb1) of
  // the K range read B from it at k = (kb - b2_kb0) * 64 (+ b2_lo_off for the lo pass); k-blocks >= b2_kb1
  // read A and B at k + kjump.  The projected-context step (D5 folded into D6/D7) uses it for the
  // alpha K range, whose B rows are the context's ctx . W projections (nmt_ctx::cw).
  int b2_kb0, b2_kb1, b2_lo_off, kjump;
};

struct EpiParams {
  float* out;
  int ldc;
  const float* bias;
  float4* part;
  int n_valid;
  int n_tiles;
  size_t split_stride;
  int* cpm_out;  // EPI_LSE: runs per m-tile (partials per row = 2 * cpm), written by CTA 0
  int rows_per_split;  // EPI_STORE: row offset of split-K partial s is s * rows_per_split
  float2* topk;        // EPI_TOPK: [R][2 cpm][kTopK] (logit, column) per (row, run, half), descending
  // EPI_GRU (fused GRU gates, B rows interleaved per 32-unit group as [r | u | h~ | zero pad]):
  //   h' = u*h + (1-u)*tanh(r*acc_x + gx_x) with r = sigm(gx_r + acc_r), u = sigm(gx_u + acc_u)
  const float* gx;     // [.][gx_ld] input projections + biases, row gx_row(r): [r | u | x] blocks of Hp
  int gx_ld;
  const int* row_y;    // gx row of output row r: row_y[r] (< 0 -> y_bos)
  int y_bos;
  const int* row_src;  // previous state of output row r: S[row_src[r]]
  const float* S;      // [.][Hp]
  float* S1;           // [R][Hp] new state (fp32)
  __nv_bfloat16* X;    // [R][ldx] new state as the next GEMM's bf16 operand (lo at +lo_x if > 0)
  int ldx, lo_x, Hp;
  unsigned long long* trace;  // diagnostic builds only (NMT_GEMM_TRACE): [CTA][8] globaltimer stamps
  // EPI_GRU2 (fused decoder GRU2, B rows per 32-unit group [hx | r | u | cx], s1 . U_nl K range on the
  // first Hp columns of A, c . Wc on the rest): s2 = u*s1 + (1-u)*tanh(r*(hx + bx_nl) + cx),
  // r = sigm(acc_r + b_nl[r]), u = sigm(acc_u + b_nl[u]); input s1 = S1 (above)
  float* Sout;             // arena states [.][Hp]: s2 -> slot row_dst[r] (>= 0)
  const int* row_dst;
  const struct GrpStep* gs;  // multi-context step: per-group arenas (Sout unused), else null
  const int* row_grp;
  const float* b_nl;       // [2Hp]
  const float* bx_nl;      // [Hp]
  int x_col;               // column of s2 in X
  // EPI_READOUT (fused readout D7; BN = 128 CTA-pair tiles, no split-K): t = maxout / tanh of
  // (acc + Eproj[y]) -> arena T (slot row_dst) and the vocabulary GEMM's A operand (bias columns at E)
  const float* Eproj;      // [V + 1][ROp] (row V: BOS / dead rows)
  int V, E, Ep, maxout;
  float* Tout;             // arena t [.][Ep]
  __nv_bfloat16* A_t;      // [R][lda_t] (lo at +lo_t when > 0)
  int lda_t, lo_t;
};
constexpr int kTopK = 8;  // NMT_TOPK_MAX: words per row kept by the top-k vocabulary epilogue

CUtensorMap make_tmap_bf16(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);
void gemm_store(const CUtensorMap& a, const CUtensorMap& b, const GemmShape& g, float* out, int ldc, int out_rows,
                const float* bias, int M_max, cudaStream_t st, size_t split_stride = 0);
void gemm_store256(const CUtensorMap& a, const CUtensorMap& b, const GemmShape& g, float* out, int ldc, int out_rows,
                   const float* bias, int M_max, cudaStream_t st, size_t split_stride = 0);
// out[r][c] = bias[c] + sum_s part[s * stride + r * ldc + c]  (fixed order: deterministic)
void splitk_reduce(const float* part, int ksplit, size_t stride, int M, int N, int ldc, const float* bias, float* out,
                   cudaStream_t st, __nv_bfloat16* out16 = nullptr);
// the same for the attention keys: also out_e = exp(2 out) with the exponent clamped to +-kAttnExpClamp, and
// bigp |= 1 where it was clamped
// E7 pctx / exp(2 pctx) (+ b_att) from the split-K partials of the encoder's GEMM ctx . Wcat^T (columns < Cp)
// and, when cw != null, the projected-context B operands cw[NW][2 Apad] (columns Cp.. transposed; bf16 hi | lo,
// zero past Tx); Apad and NW multiples of 32
constexpr int kEncSplit = 5;
void enc_proj_reduce(const float* part, int ksplit, size_t stride, int Tx, int ldc, int Cp, const float* bias,
                     float* pctx, float* epctx, int* bigp, int NW, int Apad, bool split, __nv_bfloat16* cw,
                     cudaStream_t st);
void splitk_reduce_pctx(const float* part, int ksplit, size_t stride, int M, int N, int ldc, const float* bias,
                        float* out, float* out_e, int* bigp, cudaStream_t st);
void gemm_store_pair(const CUtensorMap& a, const CUtensorMap& b_half, const GemmShape& g, float* out, int ldc,
                     int out_rows, const float* bias, int M_max, cudaStream_t st, size_t split_stride = 0);
void gemm_topk_pair(const CUtensorMap& a, const CUtensorMap& b_half, const GemmShape& g, float2* topk, int n_valid,
                    cudaStream_t st, int* cpm_out);
void gemm_lse_pair(const CUtensorMap& a, const CUtensorMap& b_half, const GemmShape& g, float4* part, int n_valid,
                   cudaStream_t st, int* cpm_out);
// GEMM s.[U|Ux] with the GRU gates fused into the epilogue (CTA pairs, no split-K); see EPI_GRU
void gemm_store_pair128(const CUtensorMap& a, const CUtensorMap& b_q, const GemmShape& g, float* out, int ldc,
                        int out_rows, const float* bias, int M_max, cudaStream_t st, size_t split_stride = 0);
void gemm_gru_pair(const CUtensorMap& a, const CUtensorMap& b_half, const GemmShape& g, const EpiParams& ep, int M_max,
                   cudaStream_t st);
// GEMM [s1 | c] . W_g2 (interleaved per 32-unit group [hx | r | u | cx]) with the decoder's GRU2 fused
// into the epilogue (EPI_GRU2; CTA pairs, no split-K, no partials).  `b2`: the projected-context step's
// second B operand (the context's ctx.[Wc|Wcx] rows for the alpha K range, GemmShape.b2_kb0/1), or null
void gemm_gru2_pair(const CUtensorMap& a, const CUtensorMap& b_half, const GemmShape& g, const EpiParams& ep, int M_max,
                    cudaStream_t st, const CUtensorMap* b2 = nullptr);
// GEMM [c | s2] . [W_ctx; W_l] with the readout (maxout or tanh over + Eproj[y]) fused into the epilogue
// (EPI_READOUT; CTA pairs with 256 x 128 tiles, `b_q` = W_ro map with a 64-row box, no split-K); `b2` as
// for gemm_gru2_pair (the context's ctx.W_ctx rows)
void gemm_readout_pair(const CUtensorMap& a, const CUtensorMap& b_q, const GemmShape& g, const EpiParams& ep, int M_max,
                       cudaStream_t st, const CUtensorMap* b2 = nullptr);
void gemm_readout_pair64(const CUtensorMap& a, const CUtensorMap& b_e, const GemmShape& g, const EpiParams& ep,
                         int M_max, cudaStream_t st, const CUtensorMap* b2 = nullptr);
void gemm_lse(const CUtensorMap& a, const CUtensorMap& b, const GemmShape& g, float4* part, int n_valid, int M_max,
              cudaStream_t st, int* cpm_out);

inline GemmShape gemm_shape(int M, const int* M_dev, int N, int K, int a_col0, bool split, int a_lo_off,
                            int b_lo_off) {
  GemmShape g{};
  g.M = M;
  g.M_dev = M_dev;
  g.N = N;
  g.a_col0 = a_col0;
  g.a_lo_off = a_lo_off;
  g.b_lo_off = b_lo_off;
  g.passes = split ? 3 : 1;
  g.nreg = 1;
  g.reg_n_end[0] = N;
  g.reg_k0[0] = 0;
  g.reg_k1[0] = K;
  g.ksplit = 1;
  g.b_panel_rows = 0;
  g.n_off = 0;
  return g;
}
inline int gemm_ks(const GemmShape& g, int r) { return g.reg_ks[r] > 0 ? g.reg_ks[r] : g.ksplit; }
inline int gemm_ks_max(const GemmShape& g) {
  int k = 1;
  for (int r = 0; r < g.nreg; ++r) k = k > gemm_ks(g, r) ? k : gemm_ks(g, r);
  return k;
}

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

}  // namespace nmt
