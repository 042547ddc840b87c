// kernels.cu - non-GEMM kernels of the decoder step, the device-side state cache (planner),
// the bidirectional-GRU encoder and load-time weight packing.
//
// Model equations (DL4MT/Nematus cGRU; PAPER.md:13, :30 name the model, SURVEY §8(c) writes them
// out; DESIGN.md §2 lists the readings A1-A24):
//   GRU(x,h):  [r|u] = sigm(xW + b + hU);  h~ = tanh(r*(hUx) + xWx + bx);  h' = u*h + (1-u)*h~
//   step:      s1 = GRU1(e, s);  a_j = tanh(pctx_j + s1 W_comb_att).U_att + c_tt;  alpha = softmax_j(a)
//              c = sum_j alpha_j ctx_j;  [r2|u2] = sigm(s1 U_nl + b_nl + c Wc)
//              s2 = u2*s1 + (1-u2)*tanh(r2*(s1 Ux_nl + bx_nl) + c Wcx)
//              t  = tanh(s2 W_l + e W_p + c W_ctx + b)   |  maxout pairs (2k, 2k+1)
//              log p(w) = t.W_o[:,w] + b_o[w] - logsumexp_v(t W_o + b_o)
// Device layouts: hidden dims padded to Hp = roundup(H,128), context dims to
// Cp = 2 Hp with cmap(i) = i < H ? i : Hp + i - H, embedding/readout width to Ep = roundup(E+2,64).
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"
#include "stepops.cuh"

namespace nmt {

NMT_DEV int cmap_(int i, int H, int Hp) { return i < H ? i : Hp + (i - H); }

NMT_DEV void store_split(__nv_bfloat16* hi_ptr, int lo_off, float x) {
  __nv_bfloat16 h, l;
  split_bf16(x, h, l);
  hi_ptr[0] = h;
  if (lo_off > 0) hi_ptr[lo_off] = l;
}

// ===================================================================================== packing
// dst[rowmap(n)][col0 + kmap(k)] = split(src[k * ld_src + n])  (transpose-pack a [K x N] matrix
// into an N x K K-major bf16 operand; lo half at +lo_off columns if lo_off > 0)
__global__ void k_pack_T(const float* __restrict__ src, int ld_src, int K, int N, __nv_bfloat16* dst, int ld_dst,
                         int row0, int col0, int rmap, int kmap, int H, int Hp, int lo_off) {
  pdl_enter();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)K * N) return;
  const int k = (int)(idx / N), n = (int)(idx % N);
  const int r = row0 + (rmap ? cmap_(n, H, Hp) : n);
  const int c = col0 + (kmap ? cmap_(k, H, Hp) : k);
  store_split(dst + (int64_t)r * ld_dst + c, lo_off, src[(int64_t)k * ld_src + n]);
}
void pack_T(const float* src, int ld_src, int K, int N, __nv_bfloat16* dst, int ld_dst, int row0, int col0, int rmap,
            int kmap, int H, int Hp, int lo_off, cudaStream_t st) {
  const int64_t n = (int64_t)K * N;
  if (!n) return;
  launch_pdl(k_pack_T, (unsigned)((n + 255) / 256), 256, 0, st, src, ld_src, K, N, dst, ld_dst, row0, col0, rmap, kmap, H, Hp,
                                                        lo_off);
  CK_LAUNCH();
}

// dst[r][col0 + k] = split(src[r * ld_src + k]) for r < rows, k < K (row-major copy)
__global__ void k_pack_rows(const float* __restrict__ src, int ld_src, int rows, int K, __nv_bfloat16* dst,
                            int ld_dst, int col0, int lo_off) {
  pdl_enter();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)rows * K) return;
  const int r = (int)(idx / K), k = (int)(idx % K);
  store_split(dst + (int64_t)r * ld_dst + col0 + k, lo_off, src[(int64_t)r * ld_src + k]);
}
void pack_rows(const float* src, int ld_src, int rows, int K, __nv_bfloat16* dst, int ld_dst, int col0, int lo_off,
               cudaStream_t st) {
  const int64_t n = (int64_t)rows * K;
  if (!n) return;
  launch_pdl(k_pack_rows, (unsigned)((n + 255) / 256), 256, 0, st, src, ld_src, rows, K, dst, ld_dst, col0, lo_off);
  CK_LAUNCH();
}

// row-major bf16 [rows][cols] -> k-block panels [cols/64][rows][64] (contiguous TMA boxes)
__global__ void k_to_panels(const __nv_bfloat16* __restrict__ src, int rows, int cols, __nv_bfloat16* dst) {
  pdl_enter();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)rows * cols) return;
  const int r = (int)(idx / cols), k = (int)(idx % cols);
  dst[((int64_t)(k / 64) * rows + r) * 64 + (k % 64)] = src[idx];
}
void to_panels(const __nv_bfloat16* src, int rows, int cols, __nv_bfloat16* dst, cudaStream_t st) {
  const int64_t n = (int64_t)rows * cols;
  launch_pdl(k_to_panels, (unsigned)((n + 255) / 256), 256, 0, st, src, rows, cols, dst);
  CK_LAUNCH();
}

// fp32 [K x N] -> fp32 [N x ld_dst] transposed (W_o columns as contiguous per-word rows)
__global__ void k_transpose_f32(const float* __restrict__ src, int K, int N, float* dst, int ld_dst) {
  pdl_enter();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)K * N) return;
  const int k = (int)(idx / N), n = (int)(idx % N);
  dst[(int64_t)n * ld_dst + k] = src[idx];
}
void transpose_f32(const float* src, int K, int N, float* dst, int ld_dst, cudaStream_t st) {
  const int64_t n = (int64_t)K * N;
  launch_pdl(k_transpose_f32, (unsigned)((n + 255) / 256), 256, 0, st, src, K, N, dst, ld_dst);
  CK_LAUNCH();
}

// split-K partial sums -> output (+bias), in fixed split order
__global__ void k_splitk_reduce(const float* __restrict__ part, int ksplit, size_t stride, int M, int N, int ldc,
                                const float* __restrict__ bias, float* out, __nv_bfloat16* out16) {
  pdl_enter();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)M * N) return;
  const int r = (int)(i / N), c = (int)(i % N);
  float s = bias ? bias[c] : 0.f;
  for (int k = 0; k < ksplit; ++k) s += part[k * stride + (size_t)r * ldc + c];
  out[(size_t)r * ldc + c] = s;
  if (out16) out16[(size_t)r * ldc + c] = __float2bfloat16_rn(s);
}
void splitk_reduce(const float* part, int ksplit, size_t stride, int M, int N, int ldc, const float* bias, float* out,
                   cudaStream_t st, __nv_bfloat16* out16) {
  const int64_t n = (int64_t)M * N;
  if (n <= 0) return;
  launch_pdl(k_splitk_reduce, (unsigned)((n + 255) / 256), 256, 0, st, part, ksplit, stride, M, N, ldc, bias, out, out16);
  CK_LAUNCH();
}

// exp(2 x) with the exponent clamped (attention keys/queries, D4: tanh(p + q) = 1 - 2 / (1 + e^2p e^2q));
// returns whether it was clamped
NMT_DEV float exp2x_clamped(float x, bool& big) {
  const float y = 2.f * x;
  big = fabsf(y) > kAttnExpClamp;
  return expf(fminf(fmaxf(y, -kAttnExpClamp), kAttnExpClamp));
}
__global__ void k_splitk_reduce_pctx(const float* __restrict__ part, int ksplit, size_t stride, int M, int N, int ldc,
                                     const float* __restrict__ bias, float* out, float* out_e, int* bigp) {
  pdl_enter();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)M * N) return;
  const int r = (int)(i / N), c = (int)(i % N);
  float s = bias ? bias[c] : 0.f;
  for (int k = 0; k < ksplit; ++k) s += part[k * stride + (size_t)r * ldc + c];
  out[(size_t)r * ldc + c] = s;
  bool big;
  out_e[(size_t)r * ldc + c] = exp2x_clamped(s, big);
  if (big) atomicOr(bigp, 1);
}
void splitk_reduce_pctx(const float* part, int ksplit, size_t stride, int M, int N, int ldc, const float* bias,
                        float* out, float* out_e, int* bigp, cudaStream_t st) {
  const int64_t n = (int64_t)M * N;
  if (n <= 0) return;
  launch_pdl(k_splitk_reduce_pctx, (unsigned)((n + 255) / 256), 256, 0, st, part, ksplit, stride, M, N, ldc, bias, out,
             out_e, bigp);
  CK_LAUNCH();
}

// E7 + projected-context operands in one pass over the split-K partials of the encoder's single GEMM
// ctx . [Wc_att ; W_g2i c rows ; W_ro c rows]^T  (partials [ks][Tx..][ldc], ldc = Cp + NW):
//   blocks [0, nb_p): pctx = sum + b_att and exp(2 pctx) (clamped, CNT_BIGP flag) for columns < Cp;
//   blocks [nb_p, ..): 32 x 32 tiles of the remaining NW columns, transposed through shared memory into the
//   B-operand rows cw[n][j] (bf16 hi at j, lo at Apad + j; zero for Tx <= j < Apad) of the D6 / D7 GEMMs'
//   alpha K range (D5 folded into D6 / D7, nmt_ctx::cw).
__global__ void __launch_bounds__(256) k_enc_proj_reduce(const float* __restrict__ part, int ksplit, size_t stride,
                                                         int Tx, int ldc, int Cp, const float* __restrict__ bias,
                                                         float* pctx, float* epctx, int* bigp, int nb_p, int NW,
                                                         int Apad, int split, __nv_bfloat16* __restrict__ cw) {
  pdl_enter();
  if ((int)blockIdx.x < nb_p) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)Tx * Cp) return;
    const int r = (int)(i / Cp), c = (int)(i % Cp);
    float s = bias[c];
    for (int k = 0; k < ksplit; ++k) s += part[k * stride + (size_t)r * ldc + c];
    pctx[(size_t)r * Cp + c] = s;
    bool big;
    epctx[(size_t)r * Cp + c] = exp2x_clamped(s, big);
    if (big) atomicOr(bigp, 1);
    return;
  }
  __shared__ float tile[32][33];
  const int t = blockIdx.x - nb_p, tj = Apad / 32;
  const int n0 = (t / tj) * 32, j0 = (t % tj) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 32 per pass
  for (int jj = ty; jj < 32; jj += 8) {  // coalesced along the partials' columns n
    const int j = j0 + jj;
    float s = 0.f;
    if (j < Tx)
      for (int k = 0; k < ksplit; ++k) s += part[k * stride + (size_t)j * ldc + Cp + n0 + tx];
    tile[jj][tx] = s;
  }
  __syncthreads();
  for (int nn = ty; nn < 32; nn += 8) {  // coalesced along the B-operand rows' token columns j
    const float v = tile[tx][nn];
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    __nv_bfloat16* row = cw + (size_t)(n0 + nn) * 2 * Apad + j0 + tx;
    row[0] = hi;
    row[Apad] = __float2bfloat16_rn(split ? v - __bfloat162float(hi) : 0.f);
  }
}
void enc_proj_reduce(const float* part, int ksplit, size_t stride, int Tx, int ldc, int Cp, const float* bias,
                     float* pctx, float* epctx, int* bigp, int NW, int Apad, bool split, __nv_bfloat16* cw,
                     cudaStream_t st) {
  const int nb_p = (int)(((int64_t)Tx * Cp + 255) / 256);
  const int nb_w = cw ? (NW / 32) * (Apad / 32) : 0;
  launch_pdl(k_enc_proj_reduce, (unsigned)(nb_p + nb_w), 256, 0, st, part, ksplit, stride, Tx, ldc, Cp, bias, pctx,
             epctx, bigp, nb_p, NW, Apad, (int)split, cw);
  CK_LAUNCH();
}

// ===================================================================================== planner
// Device-side state cache (SURVEY §8(a) D0; PAPER.md:109 "collapsed edges", :121 "Cache state
// pointers and probabilities at target nodes").  Keys (parent, word) -> child id in an open-
// addressing table; child ids are assigned in first-appearance order of the request stream.
constexpr int64_t KEY_EMPTY = -1;
constexpr int VAL_INIT = INT32_MIN;

NMT_DEV uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

NMT_DEV int hash_insert(unsigned long long* keys, uint64_t mask, int64_t key) {
  uint64_t h = mix64((uint64_t)key) & mask;
  while (true) {
    const unsigned long long prev = atomicCAS(&keys[h], (unsigned long long)KEY_EMPTY, (unsigned long long)key);
    if (prev == (unsigned long long)KEY_EMPTY || prev == (unsigned long long)key) return (int)h;
    h = (h + 1) & mask;
  }
}

constexpr int kPlanSmemOffsets = 8192;  // offsets staged in shared memory up to this many parents
__global__ void k_plan_intern(CtxDev c, PlanIO io, const PlanDesc* __restrict__ gd) {
  pdl_enter();
  if (gd) {  // multi-context call: this block row serves group blockIdx.y
    c = gd[blockIdx.y].c;
    io = gd[blockIdx.y].io;
  }
  __shared__ int soff[kPlanSmemOffsets + 1];
  const bool use_smem = io.n_par + 1 <= kPlanSmemOffsets + 1;
  const int* offs = io.offsets;
  if (use_smem) {
    for (int k = threadIdx.x; k <= io.n_par; k += blockDim.x) soff[k] = io.offsets[k];
    __syncthreads();
    offs = soff;
  }
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n_nodes = c.counters[CNT_NODES];
  if (i < io.n_cand) {
    int lo = 0, hi = io.n_par;  // find k with offsets[k] <= i < offsets[k+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (offs[mid] <= i) lo = mid; else hi = mid;
    }
    const int k = lo;
    io.cand_k[i] = k;
    const int p = io.parents[k], w = io.words[i];
    int slot = -1;
    if (p < 0 || p >= n_nodes) {
      atomicOr(&c.counters[CNT_ERR], ERR_BAD_STATE);
    } else if (w < 0 || w >= c.V) {
      atomicOr(&c.counters[CNT_ERR], ERR_TOKEN);
    } else {
      slot = hash_insert(c.hkeys, c.hmask, ((int64_t)p << 32) | (uint32_t)w);
      atomicMax(&c.hvals[slot], -2 - i);
    }
    io.cand_hslot[i] = slot;
  }
  if (i < io.n_par) {
    const int p = io.parents[i];
    const int o0 = offs[i], o1 = offs[i + 1];
    if (o1 < o0) atomicOr(&c.counters[CNT_ERR], ERR_OFFSETS);
    if (p < 0 || p >= n_nodes) atomicOr(&c.counters[CNT_ERR], ERR_BAD_STATE);
    else if (o1 > o0 || io.step_all) atomicMin(&c.node_claim[p], i);
  }
}

// block-wide exclusive scan of one int per thread (1024 threads); returns the total
NMT_DEV int block_scan_excl(int v, int* smem32, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem32[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int s = lane < (int)(blockDim.x >> 5) ? smem32[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    smem32[lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  const int warp_prefix = warp ? smem32[warp - 1] : 0;
  total = smem32[(blockDim.x >> 5) - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

// Multi-CTA assignment (blocks [0, Bc) = candidates, [Bc, Bc + Bp) = parents, 256 threads each):
//  k_plan_flags : first-appearance flags of new (parent, word) keys / parents that must be stepped,
//                 one count per block, and a snapshot of the node/slot counters;
//  k_plan_assign: block prefix from the counts + in-block scan -> node ids in first-appearance
//                 order (deterministic), row list of the parents to step (in request order).
constexpr int kPlanBlock = 256;
NMT_DEV int block_count(int v, int* red) {  // sum over a 256-thread block
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = __reduce_add_sync(0xffffffffu, v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int t = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
  return t;
}
__global__ void __launch_bounds__(kPlanBlock) k_plan_flags(CtxDev c, PlanIO io, int Bc, const PlanDesc* __restrict__ gd) {
  pdl_enter();
  __shared__ int red[8];
  const int b = blockIdx.x;
  if (gd) {
    c = gd[blockIdx.y].c;
    io = gd[blockIdx.y].io;
    Bc = (io.n_cand + kPlanBlock - 1) / kPlanBlock;
    if (b >= Bc + max(1, (io.n_par + kPlanBlock - 1) / kPlanBlock)) return;
  }
  int f = 0;
  if (b < Bc) {
    const int i = b * kPlanBlock + threadIdx.x;
    if (i < io.n_cand) {
      const int hs = io.cand_hslot[i];
      f = hs >= 0 && c.hvals[hs] == -2 - i;
      io.cflag[i] = f;
    }
  } else {
    const int k = (b - Bc) * kPlanBlock + threadIdx.x;
    const int n_nodes0 = c.counters[CNT_NODES];
    if (k < io.n_par) {
      const int p = io.parents[k];
      f = p >= 0 && p < n_nodes0 && (io.step_all || io.offsets[k + 1] > io.offsets[k]) && c.node_slot[p] < 0 &&
          c.node_claim[p] == k;
      io.pflag[k] = f;
    }
  }
  const int t = block_count(f, red);
  if (threadIdx.x == 0) {
    io.bcount[b] = t;
    if (b == 0) {
      io.snap[0] = c.counters[CNT_NODES];
      io.snap[1] = c.counters[CNT_SLOTS];
    }
  }
}

__global__ void __launch_bounds__(kPlanBlock) k_plan_assign(CtxDev c, PlanIO io, int Bc, int Bp, int* R_out,
                                                            const PlanDesc* __restrict__ gd) {
  pdl_enter();
  __shared__ int red[32];
  const int b = blockIdx.x;
  if (gd) {
    c = gd[blockIdx.y].c;
    io = gd[blockIdx.y].io;
    R_out = gd[blockIdx.y].R_out;
    Bc = (io.n_cand + kPlanBlock - 1) / kPlanBlock;
    Bp = max(1, (io.n_par + kPlanBlock - 1) / kPlanBlock);
    if (b >= Bc + Bp) return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool cand = b < Bc;
  const int b0 = cand ? 0 : Bc, bi = cand ? b : b - Bc;
  // prefix of the earlier blocks of the same kind (warp 0), totals (block 0 only)
  if (warp == 0) {
    int pre = 0;
    for (int q = lane; q < bi; q += 32) pre += io.bcount[b0 + q];
    pre = __reduce_add_sync(0xffffffffu, pre);
    if (lane == 0) red[16] = pre;
    if (b == 0) {
      int tc = 0, tp = 0;
      for (int q = lane; q < Bc; q += 32) tc += io.bcount[q];
      for (int q = lane; q < Bp; q += 32) tp += io.bcount[Bc + q];
      tc = __reduce_add_sync(0xffffffffu, tc);
      tp = __reduce_add_sync(0xffffffffu, tp);
      if (lane == 0) {
        c.counters[CNT_NODES] = io.snap[0] + tc;
        c.counters[CNT_SLOTS] = io.snap[1] + tp;
        *R_out = tp;
      }
    }
  }
  const int e = bi * kPlanBlock + threadIdx.x;
  const int n = cand ? io.n_cand : io.n_par;
  const int f = e < n ? (cand ? io.cflag[e] : io.pflag[e]) : 0;
  // in-block exclusive scan
  int x = f;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) red[warp] = x;
  __syncthreads();
  int wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += red[w];
  const int pos = red[16] + wpre + x - f;
  if (cand) {
    if (f) {
      const int id = io.snap[0] + pos;
      const int k = io.cand_k[e];
      c.node_word[id] = io.words[e];
      c.node_parent[id] = io.parents[k];
      c.node_slot[id] = -1;
      c.node_claim[id] = INT32_MAX;
      c.hvals[io.cand_hslot[e]] = id;
    }
  } else if (e < n) {
    const int p = io.parents[e];
    if (f) {
      const int r = pos;
      const int par = c.node_parent[p];
      io.row_src[r] = par >= 0 ? c.node_slot[par] : c.node_src[p];  // parents stepped in earlier calls
      io.row_y[r] = c.node_word[p];
      io.row_dst[r] = io.snap[1] + r;
      io.row_node[r] = p;
      c.node_slot[p] = io.snap[1] + r;
    }
    if (p >= 0 && p < io.snap[0]) c.node_claim[p] = INT32_MAX;  // release claims
  }
}

void plan(const CtxDev& c, const PlanIO& io, int* R_dev, cudaStream_t st) {
  const int n = io.n_cand > io.n_par ? io.n_cand : io.n_par;
  const PlanDesc* none = nullptr;
  if (n > 0) {
    launch_pdl(k_plan_intern, (n + 255) / 256, 256, 0, st, c, io, none);
    CK_LAUNCH();
  }
  const int Bc = (io.n_cand + kPlanBlock - 1) / kPlanBlock, Bp = (io.n_par + kPlanBlock - 1) / kPlanBlock;
  const int B = Bc + Bp > 0 ? Bc + Bp : 1;
  launch_pdl(k_plan_flags, B, kPlanBlock, 0, st, c, io, Bc, none);
  CK_LAUNCH();
  launch_pdl(k_plan_assign, B, kPlanBlock, 0, st, c, io, Bc, Bp, R_dev, none);
  CK_LAUNCH();
}
void plan_multi(const PlanDesc* descs, int G, int max_cand, int max_par, cudaStream_t st) {
  const CtxDev c{};
  const PlanIO io{};
  const int n = std::max(max_cand, max_par);
  if (n > 0) {
    launch_pdl(k_plan_intern, dim3((n + 255) / 256, G), 256, 0, st, c, io, descs);
    CK_LAUNCH();
  }
  const int B = (max_cand + kPlanBlock - 1) / kPlanBlock + std::max(1, (max_par + kPlanBlock - 1) / kPlanBlock);
  launch_pdl(k_plan_flags, dim3(B, G), kPlanBlock, 0, st, c, io, 0, descs);
  CK_LAUNCH();
  int* no_r = nullptr;
  launch_pdl(k_plan_assign, dim3(B, G), kPlanBlock, 0, st, c, io, 0, 0, no_r, descs);
  CK_LAUNCH();
}

// rehash all entries of an old table into a new (larger) one
__global__ void k_rehash(const unsigned long long* okeys, const int* ovals, int64_t ocap, unsigned long long* nkeys,
                         int* nvals, uint64_t nmask) {
  pdl_enter();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ocap) return;
  const int64_t key = (int64_t)okeys[i];
  if (key == KEY_EMPTY) return;
  const int s = hash_insert(nkeys, nmask, key);
  nvals[s] = ovals[i];
}
void rehash(const unsigned long long* okeys, const int* ovals, int64_t ocap, unsigned long long* nkeys, int* nvals,
            uint64_t nmask, cudaStream_t st) {
  launch_pdl(k_rehash, (unsigned)((ocap + 255) / 256), 256, 0, st, okeys, ovals, ocap, nkeys, nvals, nmask);
  CK_LAUNCH();
}

__global__ void k_fill_i32(int* p, int64_t n, int v) {
  pdl_enter();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}
void fill_i32(int* p, int64_t n, int v, cudaStream_t st) {
  if (n <= 0) return;
  launch_pdl(k_fill_i32, (unsigned)((n + 255) / 256), 256, 0, st, p, n, v);
  CK_LAUNCH();
}

// checkpoint averaging: acc += x in fp64 (member order), out = fp32(acc / n)
__global__ void k_avg_accum(double* __restrict__ acc, const float* __restrict__ x, int64_t n, int first) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) acc[i] = first ? (double)x[i] : acc[i] + (double)x[i];
}
__global__ void k_avg_finish(float* __restrict__ out, const double* __restrict__ acc, int64_t n, double members) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (float)(acc[i] / members);
}
void avg_accum(double* acc, const float* x, int64_t n, bool first, cudaStream_t st) {
  k_avg_accum<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(acc, x, n, first ? 1 : 0);
  CK_LAUNCH();
}
void avg_finish(float* out, const double* acc, int64_t n, int members, cudaStream_t st) {
  k_avg_finish<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, acc, n, (double)members);
  CK_LAUNCH();
}

// context (re)initialisation for nmt_encode, one launch: the hash table is emptied, the counters and
// the root node 0 = (s0, BOS) (word -1, parent -1, state in slot 0, not stepped) are written
__global__ void k_ctx_reset(CtxDev c, int64_t hcap) {
  pdl_enter();
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = i0; i < hcap; i += (int64_t)gridDim.x * blockDim.x) {
    c.hkeys[i] = ~0ull;
    c.hvals[i] = INT32_MIN;
  }
  if (i0 == 0) {
    c.counters[CNT_NODES] = 1;
    c.counters[CNT_SLOTS] = 2;  // slot 0 = s0, slot 1 = scratch
    c.counters[CNT_ERR] = 0;
    c.counters[CNT_R] = 0;
    c.counters[CNT_BIGP] = 0;
    c.node_word[0] = -1;
    c.node_parent[0] = -1;
    c.node_src[0] = 0;
    c.node_slot[0] = -1;
  }
}
void ctx_reset(const CtxDev& c, int64_t hcap, cudaStream_t st) {
  const int64_t b = std::min<int64_t>((hcap + 255) / 256, 4 * kNumSMs);
  launch_pdl(k_ctx_reset, (unsigned)std::max<int64_t>(b, 1), 256, 0, st, c, hcap);
  CK_LAUNCH();
}

// inject parentless nodes with their own input slots (synthetic parents for bench/tests); the last
// block to finish publishes the new node/slot counts (every block has read them by then)
__global__ void k_inject(CtxDev c, int n, const float* s, const int* y, int* out_ids, int* done) {
  pdl_enter();
  const int n_nodes0 = c.counters[CNT_NODES], n_slots0 = c.counters[CNT_SLOTS];
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int slot = n_slots0 + i;
    for (int j = threadIdx.x; j < c.H; j += blockDim.x) c.S[(int64_t)slot * c.Hp + j] = s[(int64_t)i * c.H + j];
    if (threadIdx.x == 0) {
      const int id = n_nodes0 + i;
      int yy = y[i];
      if (yy < -1 || yy >= c.V) {
        atomicOr(&c.counters[CNT_ERR], ERR_TOKEN);
        yy = -1;
      }
      c.node_word[id] = yy;
      c.node_parent[id] = -1;
      c.node_src[id] = slot;
      c.node_slot[id] = -1;
      c.node_claim[id] = INT32_MAX;
      out_ids[i] = id;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done, 1) == (int)gridDim.x - 1) {
      c.counters[CNT_NODES] = n_nodes0 + n;
      c.counters[CNT_SLOTS] = n_slots0 + n;
      *done = 0;
    }
  }
}
void inject(const CtxDev& c, int n, const float* s, const int* y, int* out_ids, int* done, cudaStream_t st) {
  launch_pdl(k_inject, n < 1024 ? n : 1024, 256, 0, st, c, n, s, y, out_ids, done);
  CK_LAUNCH();
}

// ===================================================================================== step D1-D7
// Elementwise step kernels (helpers in stepops.cuh).
NMT_DEV void prefetch_l2(const void* p, uint32_t bytes) {  // TMA-unit bulk prefetch into L2 (16-byte granules)
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__global__ void k_gather_state(StepDev d, const float* __restrict__ S) {
  pdl_enter();
  const int H4 = (d.H + 3) / 4;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = idx / H4, j = (idx % H4) * 4;
  if (r >= *d.R) return;
  if (j == 0 && d.row_dst[r] >= 0) {  // the row's embedding projections, read by the GRU1 epilogue and the
    const int y = d.row_y[r];          // readout: fetched into L2 now, under the GRU1 GEMM's main loop
    const int64_t yr = y < 0 ? d.V : y;
    prefetch_l2(d.Ex + yr * 3 * d.Hp, (uint32_t)(3 * d.Hp * sizeof(float)));
    prefetch_l2(d.Eproj + yr * d.ROp, (uint32_t)(d.ROp * sizeof(float)));
  }
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);  // dead rows of a multi-context step: zeros
  if (d.row_dst[r] >= 0) v = ld4((d.gs ? d.gs[d.row_grp[r]].S : S) + (int64_t)d.row_src[r] * d.Hp + j);
  store_split4(d.A_s + (int64_t)r * d.lda_s + j, d.lo_s, v);
}

// D2: GRU1 gates.  G1 = s.[U|Ux] (GEMM), Ex[y] = e.[W|Wx] + [b|bx] (precomputed per word).
__global__ void k_gru1(StepDev d, const float* __restrict__ S) {
  pdl_enter();
  const int Hp = d.Hp, H4 = (d.H + 3) / 4;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = idx / H4, j = (idx % H4) * 4;
  if (r >= *d.R) return;
  const bool live = d.row_dst[r] >= 0;
  const int y = live ? d.row_y[r] : -1;
  const float* g = d.G1 + (int64_t)r * 3 * Hp + j;
  const float* ex = d.Ex + (int64_t)(y < 0 ? d.V : y) * 3 * Hp + j;
  const float4 gr = ld4_sum(g, d.ks_g1, d.ps_g1), gu = ld4_sum(g + Hp, d.ks_g1, d.ps_g1),
               gc = ld4_sum(g + 2 * Hp, d.ks_g1, d.ps_g1);
  const float4 er = ld4(ex), eu = ld4(ex + Hp), ec = ld4(ex + 2 * Hp);
  const float4 sv = live ? ld4((d.gs ? d.gs[d.row_grp[r]].S : S) + (int64_t)d.row_src[r] * Hp + j)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 o;
#define NMT_GRU1(c) { const float rg = sigm(er.c + gr.c), ug = sigm(eu.c + gu.c); \
                      o.c = ug * sv.c + (1.f - ug) * tanhf(rg * gc.c + ec.c); }
  NMT_GRU1(x) NMT_GRU1(y) NMT_GRU1(z) NMT_GRU1(w)
#undef NMT_GRU1
  st4(d.S1 + (int64_t)r * Hp + j, o);
  store_split4(d.X + (int64_t)r * d.ldx + j, d.lo_x, o);
}

// D4+D5: MLP attention energies (MUFU tanh), softmax over source positions, context vector.
// One CTA = RPB rows of the same sentence; thread owns 8 consecutive context columns (q of its
// rows in registers).  pctx_j and ctx_j slices stream through a per-thread cp.async ring in
// shared memory (NST positions in flight).  Energies of 8 positions x RPB rows are reduced across
// the warp with a 32-value butterfly reduce-scatter (31 shuffles instead of 5 per value).
NMT_DEV void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
NMT_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
NMT_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// v[0..31] are 32 values per lane; returns sum over the warp of v[lane] (lane i gets the total of
// value i).  5 stages, 16+8+4+2+1 shuffles.
NMT_DEV float warp_reduce_scatter32(float (&v)[32], int lane) {
#pragma unroll
  for (int st = 16; st >= 1; st >>= 1) {
    const bool upper = (lane & st) != 0;
#pragma unroll
    for (int i = 0; i < st; ++i) {
      const float send = upper ? v[i] : v[i + st];
      const float keep = upper ? v[i + st] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
    }
  }
  return v[0];
}

NMT_DEV float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Energy pass of k_attention over positions [0, Tx): pctx or exp(2 pctx) slices of the thread's 8 columns
// stream through a per-thread cp.async ring.
//  tanh path (FAST = false): e_j = sum_k U_k tanh(p_jk + q_k), one SFU tanh per term.
//  exp path (FAST = true): tanh(p + q) = 1 - 2 / (1 + e^2p e^2q), so with P = e^2p (per context) and
//    Q = e^2q (per row) e_j = sum_k U_k - 2 sum_k U_k / (1 + P_jk Q_k); the constant cancels in the
//    softmax.  Two terms share one reciprocal: U/a + U'/b = (U b + U' a) / (a b), paired across the packed
//    fp32 pairs (columns c and c + 2 of the thread's 8) so every step is one FFMA2 / FMUL2.  Columns 0-3 take
//    the pair reciprocal on the FMA pipe (bit-trick seed, negated, then one cubic Newton step
//    r (1 + e + e^2), e = 1 - x r: |rel err| <= 5.1e-2 -> 1.3e-4, below tanh.approx's 2^-11), columns 4-7 on
//    the SFU (rcp.approx): half a reciprocal per term, a quarter of them on the SFU.
//    u2[0..1] = +2 U (they multiply -1/x), u2[2..3] = -2 U.
// One block of JB positions j0.. of attn_energies: partial energies e[jj * RPB + rr] of this thread's 8 columns.
// FULL (uniform): all JB positions < Tx and all RPB rows live, so the per-item checks are compiled out.
template <int RPB, bool FAST, bool FULL>
NMT_DEV void attn_block(float (&e)[32], const float* pg, int Cp, int Tx, int nr, int j0, const float2 (&q2)[RPB][4],
                        const float2 (&u2)[4], float4* mine, int rstride, int hoff) {
  constexpr int JB = RPB <= 4 ? 8 : 4;  // positions per reduce-scatter: JB x RPB <= 32 values
  constexpr int NST = 8;                // positions in flight
  const float2 one2 = make_float2(1.f, 1.f);
  const float* gnext = pg + (int64_t)(j0 + NST) * Cp;  // refills: positions j0 + NST + jj
#pragma unroll
  for (int jj = 0; jj < JB; ++jj) {
    const int j = j0 + jj;
    const int slot = JB == NST ? jj : (j0 + jj) % NST;  // (JB == NST: j0 is a multiple of NST)
    cp_async_wait<NST - 1>();
    float4* sp = mine + slot * rstride;
    const float4 n0 = sp[0], n1 = sp[hoff];
    if (j + NST < Tx) {  // refill this slot with position j + NST
      cp_async16(sp, gnext + (int64_t)jj * Cp);
      cp_async16(sp + hoff, gnext + (int64_t)jj * Cp + 4);
    }
    cp_async_commit();
    if (!FULL && j >= Tx) continue;  // (uniform: the tail of the last block of positions)
    const float2 p2[4] = {make_float2(n0.x, n0.y), make_float2(n0.z, n0.w), make_float2(n1.x, n1.y),
                          make_float2(n1.z, n1.w)};
#pragma unroll
    for (int rr = 0; rr < RPB; ++rr) {
      if (!FULL && rr >= nr) continue;
      if constexpr (FAST) {
        float2 acc;
        {  // columns (0, 2) and (1, 3): FMA-pipe reciprocal of the pair product, rn = -1 / (a b)
          const float2 d0 = fma2(p2[0], q2[rr][0], one2), d1 = fma2(p2[1], q2[rr][1], one2);
          const float2 pr = mul2(d0, d1), nu = fma2(u2[0], d1, mul2(u2[1], d0));
          const float2 r0 = make_float2(__int_as_float(0xFEF311C3u - __float_as_uint(pr.x)),
                                        __int_as_float(0xFEF311C3u - __float_as_uint(pr.y)));
          const float2 er = fma2(pr, r0, one2);
          acc = mul2(nu, fma2(r0, fma2(er, er, er), r0));
        }
        {  // columns (4, 6) and (5, 7): SFU reciprocal of the pair product
          const float2 d2 = fma2(p2[2], q2[rr][2], one2), d3 = fma2(p2[3], q2[rr][3], one2);
          const float2 pr = mul2(d2, d3), nu = fma2(u2[2], d3, mul2(u2[3], d2));
          acc = fma2(nu, make_float2(rcp_approx(pr.x), rcp_approx(pr.y)), acc);
        }
        e[jj * RPB + rr] = acc.x + acc.y;
      } else {
        float sacc = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          sacc = fmaf(tanh_approx(p2[k].x + q2[rr][k].x), u2[k].x, sacc);
          sacc = fmaf(tanh_approx(p2[k].y + q2[rr][k].y), u2[k].y, sacc);
        }
        e[jj * RPB + rr] = sacc;
      }
    }
  }
}

template <int RPB, bool FAST>
NMT_DEV void attn_energies(const float* pg, int Cp, int Tx, int nr, const float2 (&q2)[RPB][4],
                           const float2 (&u2)[4], float4* mine, int rstride, int hoff, float* red, int warp, int lane,
                           int Tx8) {
  constexpr int JB = RPB <= 4 ? 8 : 4;  // positions per reduce-scatter: JB x RPB <= 32 values
  constexpr int NST = 8;                // positions in flight
#pragma unroll
  for (int i = 0; i < NST; ++i) {
    if (i < Tx) {
      cp_async16(mine + i * rstride, pg + (int64_t)i * Cp);
      cp_async16(mine + i * rstride + hoff, pg + (int64_t)i * Cp + 4);
    }
    cp_async_commit();
  }
  for (int j0 = 0; j0 < Tx; j0 += JB) {
    float e[32];  // e[jj * RPB + rr] partial energies of positions j0..j0+JB-1 (zero padded)
#pragma unroll
    for (int i = 0; i < 32; ++i) e[i] = 0.f;
    if (j0 + JB <= Tx && nr == RPB) attn_block<RPB, FAST, true>(e, pg, Cp, Tx, nr, j0, q2, u2, mine, rstride, hoff);
    else attn_block<RPB, FAST, false>(e, pg, Cp, Tx, nr, j0, q2, u2, mine, rstride, hoff);
    const float tot = warp_reduce_scatter32(e, lane);  // lane = jj * RPB + rr
    if (lane < JB * RPB) red[(warp * RPB + lane % RPB) * Tx8 + j0 + lane / RPB] = tot;
  }
  cp_async_wait<0>();
}

// D3-D5 attention.  Rows: with a multi-context step (d.gs) CTA b takes rows [RPB b, RPB b + RPB) (groups
// start at multiples of 4); otherwise the R rows are split evenly over the grid (CTA b: rows
// [R b / G, R (b + 1) / G)), so with two CTAs per SM every SM carries the same number of rows +-1.
template <int RPB>
__global__ void __launch_bounds__(256, 2) k_attention(StepDev d, AttnCtx a) {
  pdl_enter();
  static_assert(RPB >= 1 && RPB <= 8, "rows per CTA");
  constexpr int NST = 8;
  const int R = *d.R;
  int r0, nr;
  if (d.gs) {
    r0 = blockIdx.x * RPB;
    nr = min(RPB, R - r0);
  } else {
    r0 = (int)((int64_t)R * blockIdx.x / gridDim.x);
    nr = (int)((int64_t)R * (blockIdx.x + 1) / gridDim.x) - r0;
  }
  if (nr <= 0) return;
  const int* cnt = a.counters;
  if (d.gs) {
    const GrpStep& g = d.gs[d.row_grp[r0]];
    a.pctx = g.pctx;
    a.ctx = g.ctx;
    a.Tx = g.Tx;
    a.epctx = g.epctx;
    cnt = g.counters;
  }
  const int Cp = d.Cp, Tx = a.Tx;
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = threadIdx.x * 8;
  extern __shared__ float4 smq[];
  float4* ring = smq;                                                   // [NST][blockDim][2] float4
  float* red = reinterpret_cast<float*>(ring + NST * blockDim.x * 2);  // [nw][RPB][Tx8]
  const int Tx8 = (Tx + 7) & ~7;
  float* alpha = red + nw * RPB * Tx8;                                  // [RPB][Tx]
  // ring [NST][blockDim][2] float4: a thread's two 16-byte cp.async of a position fill one 32-byte chunk
  // (measured: the [NST][2][blockDim] layout, conflict-free for the LDS.128 reads, is ~1.9x slower)
  float4* mine = ring + threadIdx.x * 2;
  const int rstride = blockDim.x * 2, hoff = 1;
  float q[RPB][8], u[8];
  bool big = a.epctx == nullptr || cnt[CNT_BIGP] != 0;
#ifdef NMT_DIAG
  big |= d.diag_attn_slow != 0;  // (diagnostic A/B: force the tanh path)
#endif
#pragma unroll
  for (int rr = 0; rr < RPB; ++rr) {
    const bool ok = rr < nr;
    const float* qp = d.Q + (int64_t)(r0 + rr) * Cp + c0;
    const float4 x0 = ok ? ld4_sum(qp, d.ks_q, d.ps_q) : make_float4(0, 0, 0, 0),
                 x1 = ok ? ld4_sum(qp + 4, d.ks_q, d.ps_q) : make_float4(0, 0, 0, 0);
    q[rr][0] = x0.x; q[rr][1] = x0.y; q[rr][2] = x0.z; q[rr][3] = x0.w;
    q[rr][4] = x1.x; q[rr][5] = x1.y; q[rr][6] = x1.z; q[rr][7] = x1.w;
#pragma unroll
    for (int k = 0; k < 8; ++k) big |= fabsf(2.f * q[rr][k]) > kAttnExpClamp;
  }
  {
    const float4* up = reinterpret_cast<const float4*>(a.U_att + c0);
    const float4 x0 = up[0], x1 = up[1];
    u[0] = x0.x; u[1] = x0.y; u[2] = x0.z; u[3] = x0.w; u[4] = x1.x; u[5] = x1.y; u[6] = x1.z; u[7] = x1.w;
  }
  // exp path unless some exponent of this CTA's rows or of the context's keys had to be clamped
  const bool fast = !__syncthreads_or(big);
  {
    float2 q2[RPB][4], u2[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float s = fast ? (k < 2 ? 2.f : -2.f) : 1.f;
      u2[k] = make_float2(s * u[2 * k], s * u[2 * k + 1]);
#pragma unroll
      for (int rr = 0; rr < RPB; ++rr)
        q2[rr][k] = fast ? make_float2(__expf(2.f * q[rr][2 * k]), __expf(2.f * q[rr][2 * k + 1]))
                         : make_float2(q[rr][2 * k], q[rr][2 * k + 1]);
    }
    if (fast) attn_energies<RPB, true>(a.epctx + c0, Cp, Tx, nr, q2, u2, mine, rstride, hoff, red, warp, lane, Tx8);
    else attn_energies<RPB, false>(a.pctx + c0, Cp, Tx, nr, q2, u2, mine, rstride, hoff, red, warp, lane, Tx8);
  }
  __syncthreads();
  const float e0 = fast ? 0.f : a.c_tt;  // (a constant shift of all energies: no effect on alpha)
  for (int rr = warp; rr < nr; rr += nw) {  // softmax over j for row rr
    float mx = -INFINITY;
    for (int j = lane; j < Tx; j += 32) {
      float ev = e0;
      for (int w = 0; w < nw; ++w) ev += red[(w * RPB + rr) * Tx8 + j];
      alpha[rr * Tx + j] = ev;
      mx = fmaxf(mx, ev);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
    for (int j = lane; j < Tx; j += 32) {
      const float ev = expf(alpha[rr * Tx + j] - mx);
      alpha[rr * Tx + j] = ev;
      sum += ev;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float inv = 1.f / sum;
    for (int j = lane; j < Tx; j += 32) {
      alpha[rr * Tx + j] *= inv;
      if (d.alpha_out) d.alpha_out[(int64_t)(r0 + rr) * d.alpha_ld + j] = alpha[rr * Tx + j];
    }
  }
  __syncthreads();
  if (d.proj_k > 0) {  // projected-context step: alpha (bf16 hi | lo, zero past Tx) is the A operand of the
                       // G2 / readout GEMMs, which multiply it with cw = ctx . W; no context pass
    const int K = d.proj_k;
    for (int i = threadIdx.x; i < nr * K; i += blockDim.x) {
      const int rr = i / K, j = i % K;
      const float v = j < Tx ? alpha[rr * Tx + j] : 0.f;
      __nv_bfloat16* xp = d.X + (int64_t)(r0 + rr) * d.ldx + d.Hp + j;
      const __nv_bfloat16 h = __float2bfloat16_rn(v);
      xp[0] = h;
      if (d.lo_x > 0) xp[d.lo_x] = __float2bfloat16_rn(v - __bfloat162float(h));
    }
    return;
  }
  // context c = sum_j alpha_j ctx_j, ctx slices through the same ring (packed fp32 pairs)
  const float* cg = a.ctx + c0;
#pragma unroll
  for (int i = 0; i < NST; ++i) {
    if (i < Tx) {
      cp_async16(mine + i * rstride, cg + (int64_t)i * Cp);
      cp_async16(mine + i * rstride + hoff, cg + (int64_t)i * Cp + 4);
    }
    cp_async_commit();
  }
  float2 cacc[RPB][4];
#pragma unroll
  for (int rr = 0; rr < RPB; ++rr)
#pragma unroll
    for (int k = 0; k < 4; ++k) cacc[rr][k] = make_float2(0.f, 0.f);
  for (int j = 0; j < Tx; ++j) {
    const int slot = j % NST;
    cp_async_wait<NST - 1>();
    const float4 x0 = mine[slot * rstride], x1 = mine[slot * rstride + hoff];
    if (j + NST < Tx) {
      cp_async16(mine + slot * rstride, cg + (int64_t)(j + NST) * Cp);
      cp_async16(mine + slot * rstride + hoff, cg + (int64_t)(j + NST) * Cp + 4);
    }
    cp_async_commit();
    const float2 cv[4] = {make_float2(x0.x, x0.y), make_float2(x0.z, x0.w), make_float2(x1.x, x1.y),
                          make_float2(x1.z, x1.w)};
#pragma unroll
    for (int rr = 0; rr < RPB; ++rr) {
      if (rr < nr) {
        const float al = alpha[rr * Tx + j];
#ifdef ATTN_CTX_SCALAR
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          cacc[rr][k].x = fmaf(al, cv[k].x, cacc[rr][k].x);
          cacc[rr][k].y = fmaf(al, cv[k].y, cacc[rr][k].y);
        }
#else
        const float2 al2 = make_float2(al, al);
#pragma unroll
        for (int k = 0; k < 4; ++k) cacc[rr][k] = fma2(al2, cv[k], cacc[rr][k]);
#endif
      }
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int rr = 0; rr < RPB; ++rr) {
    if (rr >= nr) break;
    const int r = r0 + rr;
    float4* o = reinterpret_cast<float4*>(d.Cf + (int64_t)r * Cp + c0);
    const float4 v0 = make_float4(cacc[rr][0].x, cacc[rr][0].y, cacc[rr][1].x, cacc[rr][1].y);
    const float4 v1 = make_float4(cacc[rr][2].x, cacc[rr][2].y, cacc[rr][3].x, cacc[rr][3].y);
    o[0] = v0;
    o[1] = v1;
    __nv_bfloat16* xp = d.X + (int64_t)r * d.ldx + d.Hp + c0;
    store_split4(xp, d.lo_x, v0);
    store_split4(xp + 4, d.lo_x, v1);
  }
}

// D6: GRU2 gates (gru2_elem, stepops.cuh)
__global__ void k_gru2(StepDev d, float* __restrict__ S) {
  pdl_enter();
  gru2_elem(d, S, blockIdx.x * blockDim.x + threadIdx.x);
}

// D7: readout activation (readout_elem, stepops.cuh)
__global__ void k_readout(StepDev d, float* __restrict__ T) {
  pdl_enter();
  readout_elem(d, T, blockIdx.x * blockDim.x + threadIdx.x);
}

// D9a: combine the per-run (max, sum, argmax) partials of each row in fixed column order.
__global__ void k_finalize(StepDev d, float* __restrict__ logZ, int* __restrict__ amax) {
  pdl_enter();
  const int R = *d.R;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= R) return;
  const int np = 2 * *d.cpm;  // (run, half) partials in column order
  const float4* p = d.part + (int64_t)warp * np;
  float4 v[10];  // np <= 2 * 148: all loads in flight before combining
#pragma unroll
  for (int i = 0; i < 10; ++i) v[i] = lane + 32 * i < np ? p[lane + 32 * i] : make_float4(-INFINITY, 0.f, 0.f, 0.f);
  float m = -INFINITY, s = 0.f;
  int am = 0x7fffffff;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    if (v[i].x > m) {
      s = s * expf(m - v[i].x) + v[i].y;
      m = v[i].x;
      am = __float_as_int(v[i].z);
    } else if (v[i].x > -INFINITY) {
      s += v[i].y * expf(v[i].x - m);
      if (v[i].x == m) am = min(am, __float_as_int(v[i].z));  // runs/halves interleave columns
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const int a2 = __shfl_xor_sync(0xffffffffu, am, o);
    const float mm = fmaxf(m, m2);
    const float ns = (m > -INFINITY ? s * expf(m - mm) : 0.f) + (m2 > -INFINITY ? s2 * expf(m2 - mm) : 0.f);
    int na;
    if (m2 > m) na = a2;
    else if (m > m2) na = am;
    else na = min(am, a2);
    m = mm;
    s = ns;
    am = na;
  }
  if (d.xout) {  // vocab-parallel: this rank's slice partial, combined after the all-gather
    if (lane == 0) d.xout[warp] = make_float4(m, s, __int_as_float(am), 0.f);
    return;
  }
  const int slot = d.row_dst[warp];
  if (lane == 0 && slot >= 0) {
    if (d.gs) {
      const GrpStep& g = d.gs[d.row_grp[warp]];
      g.logZ[slot] = m + logf(s);
      g.amax[slot] = am;
    } else {
      logZ[slot] = m + logf(s);
      amax[slot] = am;
    }
  }
}

// D9b: per candidate log p = t . W_o[:,w] + b_o[w] - logZ (fp32 gather-dot; also serves cache hits);
// the trailing blocks write each parent's argmax.
__global__ void k_gather_dot(CtxDev c, PlanIO io, const float* __restrict__ Wo32, const float* __restrict__ bo,
                             int Ep, float* out_logp, int* out_child32, long long* out_child64, int* out_argmax,
                             int cand_blocks, const PlanDesc* __restrict__ gd) {
  pdl_enter();
  if (gd) {  // multi-context call: group blockIdx.y, its own output slices
    const PlanDesc& g = gd[blockIdx.y];
    c = g.c;
    io = g.io;
    out_logp = g.out_logp;
    out_child32 = g.out_child;
    out_child64 = nullptr;
    out_argmax = g.out_argmax;
    if ((int)blockIdx.x >= cand_blocks && !out_argmax) return;
  }
  if ((int)blockIdx.x >= cand_blocks) {  // parents' argmax
    const int k = (blockIdx.x - cand_blocks) * blockDim.x + threadIdx.x;
    if (k >= io.n_par) return;
    const int p = io.parents[k];
    int v = -1;
    if (p >= 0 && p < c.counters[CNT_NODES]) {
      const int slot = c.node_slot[p];
      if (slot >= 0) v = c.amax[slot];
    }
    out_argmax[k] = v;
    return;
  }
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= io.n_cand) return;
  const int hs = io.cand_hslot[warp];
  if (hs < 0) {
    if (lane == 0) {
      out_logp[warp] = __int_as_float(0x7fc00000);
      if (out_child32) out_child32[warp] = -1;
      if (out_child64) out_child64[warp] = -1;
    }
    return;
  }
  const int p = io.parents[io.cand_k[warp]];
  const int slot = c.node_slot[p];
  const int w = io.words[warp];
  const float4* t = reinterpret_cast<const float4*>(c.T + (int64_t)slot * Ep);
  const float4* wo = reinterpret_cast<const float4*>(Wo32 + (int64_t)w * Ep);
  float s = 0.f;
  for (int k = lane; k < Ep / 4; k += 32) {
    const float4 a = t[k], b = wo[k];
    s = fmaf(a.x, b.x, s);
    s = fmaf(a.y, b.y, s);
    s = fmaf(a.z, b.z, s);
    s = fmaf(a.w, b.w, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    out_logp[warp] = s + bo[w] - c.logZ[slot];
    const int ch = c.hvals[hs];
    if (out_child32) out_child32[warp] = ch;
    if (out_child64) out_child64[warp] = ch;
  }
}

// ScoreBatch forest helpers: parents of depth d+1 = children of depth d gathered by edge position;
// per pair, the sum of its phrase's word log-probs along its path of edges and the final state.
__global__ void k_gather_idx(const int* __restrict__ src, const int* __restrict__ idx, int n, int* out) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = src[idx[i]];
}
void gather_idx(const int* src, const int* idx, int n, int* out, cudaStream_t st) {
  if (n <= 0) return;
  launch_pdl(k_gather_idx, (n + 255) / 256, 256, 0, st, src, idx, n, out);
  CK_LAUNCH();
}
__global__ void k_path_sum(const float* __restrict__ logp, const int* __restrict__ child, const int* __restrict__ off,
                           const int* __restrict__ pos, int n, float* out_logp, int* out_state) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s = 0.f;
  for (int k = off[i]; k < off[i + 1]; ++k) s += logp[pos[k]];  // depth order
  out_logp[i] = s;
  out_state[i] = child[pos[off[i + 1] - 1]];
}
void path_sum(const float* logp, const int* child, const int* off, const int* pos, int n, float* out_logp,
              int* out_state, cudaStream_t st) {
  if (n <= 0) return;
  launch_pdl(k_path_sum, (n + 255) / 256, 256, 0, st, logp, child, off, pos, n, out_logp, out_state);
  CK_LAUNCH();
}

// full log-prob row of one stepped slot (test export)
__global__ void k_full_row(const float* __restrict__ T, const float* __restrict__ Wo32, const float* __restrict__ bo,
                           const float* __restrict__ logZ, int slot, int Ep, int V, float* out) {
  pdl_enter();
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= V) return;
  const float* t = T + (int64_t)slot * Ep;
  const float* wo = Wo32 + (int64_t)w * Ep;
  float s = 0.f;
  for (int k = lane; k < Ep; k += 32) s = fmaf(t[k], wo[k], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[w] = s + bo[w] - logZ[slot];
}

size_t attention_smem_bytes(int Cp, int Tx, int rpb) {
  const int nthr = Cp / 8;
  const int nw = nthr / 32 > 0 ? nthr / 32 : 1;
  const int Tx8 = (Tx + 7) & ~7;  // (as in the kernel: JB divides 8)
  return (size_t)8 * nthr * 2 * sizeof(float4) + (size_t)(nw * rpb * Tx8 + rpb * Tx) * sizeof(float);
}

template <int RPB>
static void launch_attention(const StepDev& d, const AttnCtx& a, int grid, cudaStream_t st) {
  const int nthr = d.Cp / 8;
  const size_t smem = attention_smem_bytes(d.Cp, a.Tx, RPB);
  static std::atomic<size_t> attr[kMaxDevices];  // > 48 KB of dynamic shared memory needs the opt-in
  ensure_smem_attr(k_attention<RPB>, attr, smem);
  launch_pdl(k_attention<RPB>, grid, nthr, smem, st, d, a);
}

void step_elementwise(int which, const StepDev& d, const AttnCtx& a, float* S, float* T, float* logZ, int* amax,
                      int R_max, cudaStream_t st) {
  if (R_max <= 0) return;
  const int g = R_max < 4096 ? R_max : 4096;
  const int H4 = (d.H + 3) / 4;
  const unsigned gh = (unsigned)(((int64_t)R_max * H4 + 255) / 256);
  const unsigned ge = (unsigned)(((int64_t)R_max * (d.Ep / 4) + 255) / 256);
  (void)g;
  switch (which) {
    case EW_GATHER: launch_pdl(k_gather_state, gh, 256, 0, st, d, S); break;
    case EW_GRU1: launch_pdl(k_gru1, gh, 256, 0, st, d, S); break;
    case EW_ATTN: {
#ifdef NMT_DIAG
      const_cast<StepDev&>(d).diag_attn_slow = getenv("NMT_ATTN_SLOW") ? 1 : 0;
#endif
      int rpb, grid;
      if (d.gs) {  // multi-context rows: 4-row blocks must not straddle a group (groups start at multiples of 4)
        rpb = std::max(1, std::min(4, (R_max + kNumSMs - 1) / kNumSMs));
        if (rpb == 3) rpb = 4;
        grid = (R_max + rpb - 1) / rpb;
      } else {  // rows split evenly over two CTAs per SM (<= 4 rows each; more CTAs beyond 8 rows per SM)
        grid = std::min(R_max, 2 * kNumSMs);
        rpb = (R_max + grid - 1) / grid;
        if (rpb > 4) {
          rpb = 4;
          grid = (R_max + 3) / 4;
        }
      }
      switch (rpb) {
        case 1: launch_attention<1>(d, a, grid, st); break;
        case 2: launch_attention<2>(d, a, grid, st); break;
        case 3: launch_attention<3>(d, a, grid, st); break;
        default: launch_attention<4>(d, a, grid, st); break;
      }
      break;
    }
    case EW_GRU2: launch_pdl(k_gru2, gh, 256, 0, st, d, S); break;
    case EW_READOUT: launch_pdl(k_readout, ge, 256, 0, st, d, T); break;
    case EW_FINALIZE: launch_pdl(k_finalize, (R_max * 32 + 255) / 256, 256, 0, st, d, logZ, amax); break;
  }
  CK_LAUNCH();
}

// Beam step: the vocabulary operand rows of already-stepped parents, rebuilt
// from the t cached in the arena (bit-identical to what k_readout wrote when they were stepped).
__global__ void k_beam_gather(StepDev d, CtxDev c, const int* __restrict__ parents, int n) {
  pdl_enter();
  const int E4 = d.Ep / 4;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = idx / E4, k = (idx % E4) * 4;
  if (r >= n) return;
  const int p = parents[r];
  const int slot = (p >= 0) ? c.node_slot[p] : -1;
  float tp[4] = {0.f, 0.f, 0.f, 0.f};
  if (slot >= 0) {
    const float4 t4 = ld4(c.T + (int64_t)slot * d.Ep + k);
    tp[0] = t4.x; tp[1] = t4.y; tp[2] = t4.z; tp[3] = t4.w;
  } else if (k == 0) {
    atomicOr(&c.counters[CNT_ERR], ERR_BAD_STATE);
  }
  write_vocab_operand(d, r, k, tp);
}
// merge the 2 cpm (logit, column) lists of each row into its k best columns: descending logit,
// ties -> lower column (the order a single sorted scan of the row would give).  Warp per row.
__global__ void k_topk_merge(const float2* __restrict__ topk, const int* __restrict__ cpm_dev, int n, int k,
                             int* __restrict__ out_words) {
  pdl_enter();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n) return;
  const int nc = 2 * (*cpm_dev) * kTopK;
  const float2* L = topk + (size_t)row * nc;
  int taken[kTopK];
#pragma unroll
  for (int q = 0; q < kTopK; ++q) taken[q] = -1;
  for (int q = 0; q < k; ++q) {
    float bv = -INFINITY;
    int bi = INT32_MAX;
    for (int i = lane; i < nc; i += 32) {
      const float2 e = L[i];
      const int col = __float_as_int(e.y);
      bool used = false;
#pragma unroll
      for (int u = 0; u < kTopK; ++u) used |= (u < q && taken[u] == col);
      if (!used && col != INT32_MAX && (e.x > bv || (e.x == bv && col < bi))) {
        bv = e.x;
        bi = col;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
#pragma unroll
    for (int u = 0; u < kTopK; ++u)
      if (u == q) taken[u] = bi;
    if (lane == 0) out_words[(size_t)row * k + q] = bi == INT32_MAX ? 0 : bi;
  }
}
void beam_gather(const StepDev& d, const CtxDev& c, const int* parents, int n, cudaStream_t st) {
  const int64_t tot = (int64_t)n * (d.Ep / 4);
  if (tot <= 0) return;
  launch_pdl(k_beam_gather, (unsigned)((tot + 255) / 256), 256, 0, st, d, c, parents, n);
  CK_LAUNCH();
}
void topk_merge(const float2* topk, const int* cpm_dev, int n, int k, int* out_words, cudaStream_t st) {
  if (n <= 0) return;
  launch_pdl(k_topk_merge, (unsigned)((n * 32 + 255) / 256), 256, 0, st, topk, cpm_dev, n, k, out_words);
  CK_LAUNCH();
}

void gather_dot(const CtxDev& c, const PlanIO& io, const float* Wo32, const float* bo, int Ep, float* out_logp,
                int* out_child32, long long* out_child64, int* out_argmax, cudaStream_t st) {
  const int cb = (io.n_cand * 32 + 255) / 256;
  const int pb = out_argmax ? (io.n_par + 255) / 256 : 0;
  if (cb + pb == 0) return;
  const PlanDesc* none = nullptr;
  launch_pdl(k_gather_dot, cb + pb, 256, 0, st, c, io, Wo32, bo, Ep, out_logp, out_child32, out_child64, out_argmax,
             cb, none);
  CK_LAUNCH();
}
__global__ void k_shard_combine(StepDev d, const float4* __restrict__ xall, int world, int stride,
                                float* __restrict__ logZ, int* __restrict__ amax) {
  pdl_enter();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= *d.R) return;
  float m = -INFINITY, s = 0.f;
  int am = 0x7fffffff;
  for (int k = 0; k < world; ++k) {  // rank order = ascending vocabulary slices
    const float4 v = xall[(int64_t)k * stride + r];
    if (v.x > m) {
      s = (m > -INFINITY ? s * expf(m - v.x) : 0.f) + v.y;
      m = v.x;
      am = __float_as_int(v.z);
    } else if (v.x > -INFINITY) {
      s += v.y * expf(v.x - m);
    }
  }
  const int slot = d.row_dst[r];
  if (slot < 0) return;
  if (d.gs) {
    const GrpStep& g = d.gs[d.row_grp[r]];
    g.logZ[slot] = m + logf(s);
    g.amax[slot] = am;
  } else {
    logZ[slot] = m + logf(s);
    amax[slot] = am;
  }
}
void shard_combine(const StepDev& d, const float4* xall, int world, int stride, float* logZ, int* amax, int R_max,
                   cudaStream_t st) {
  launch_pdl(k_shard_combine, (R_max + 127) / 128, 128, 0, st, d, xall, world, stride, logZ, amax);
  CK_LAUNCH();
}
__global__ void k_counters_multi(const PlanDesc* __restrict__ descs, int G, int* __restrict__ out) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < G * CNT_N) out[i] = descs[i / CNT_N].c.counters[i % CNT_N];
}
void counters_multi(const PlanDesc* descs, int G, int* out, cudaStream_t st) {
  launch_pdl(k_counters_multi, (G * CNT_N + 255) / 256, 256, 0, st, descs, G, out);
  CK_LAUNCH();
}
void gather_dot_multi(const PlanDesc* descs, int G, int max_cand, int max_par, const float* Wo32, const float* bo,
                      int Ep, cudaStream_t st) {
  const int cb = (max_cand * 32 + 255) / 256;
  const int pb = (max_par + 255) / 256;
  if (cb + pb == 0) return;
  const CtxDev c{};
  const PlanIO io{};
  float* nf = nullptr;
  int* ni = nullptr;
  long long* nl = nullptr;
  launch_pdl(k_gather_dot, dim3(cb + pb, G), 256, 0, st, c, io, Wo32, bo, Ep, nf, ni, nl, ni, cb, descs);
  CK_LAUNCH();
}

void full_row(const float* T, const float* Wo32, const float* bo, const float* logZ, int slot, int Ep, int V,
              float* out, cudaStream_t st) {
  launch_pdl(k_full_row, (V * 32 + 255) / 256, 256, 0, st, T, Wo32, bo, logZ, slot, Ep, V, out);
  CK_LAUNCH();
}

// ===================================================================================== encoder
// E1-E6 in one persistent cooperative kernel (k_enc_recur2).  CTAs [0, NB) run the forward direction,
// [NB, 2NB) the backward one.  Each CTA owns UPC hidden units, two per warp: the warp keeps the units'
// columns of [U | Ux] (r, u and candidate gates) in REGISTERS for the whole sentence, so a time step reads
// no weights at all.  The dot products use packed FFMA2.  The input projections x_j.[W|Wx] + [b|bx] are
// rows of a table precomputed per source word at load (E1+E2 become a gather into shared memory).
// h_t is exchanged through global memory as 32-bit words: the fp32 value with its two low mantissa bits
// replaced by the tag (t + 1) mod 4 (a relative perturbation <= 2^-22).  A reader polls until every word
// carries the tag of the step it needs, which merges the grid-wide barrier into the data read (one L2
// round trip per step).  Double-buffered by step parity: a writer is at most one step ahead of the
// slowest reader, and the word a reader finds in its buffer is from step t, t - 2 or t - 4..., whose tags
// differ mod 4.  Each encode zeroes the words after its final grid barrier (tag 0 matches neither first
// read, tags 1 and 2), so the next encode starts clean with no reset between calls; a barrier counter that
// only grows serves the tail.
// Tail (E5): each CTA publishes the time-mean of its units, one grid barrier, then the CTAs split
// s0 = tanh(mean . W_init + b_init); their W_init rows are prefetched into shared memory at start.
// The kernel also writes the bf16 hi|lo copy of ctx (E7 input).
__device__ __forceinline__ float sigmoid_fast(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
__device__ __forceinline__ float tanh_fast(float x) {  // |err| ~ 1e-7 (not tanh.approx)
  const float e = __expf(2.f * fminf(fmaxf(x, -15.f), 15.f));
  return 1.f - __fdividef(2.f, e + 1.f);
}
constexpr int kPinMax = 512;  // sources up to this length have their input projections staged in smem
// TWO units per warp (UPC <= 16 -> <= 8 warps): the warp keeps 6 weight columns in registers (192 per
// lane, up to 255 allowed at 256 threads), so only UPC / 2 warps read h from shared memory each step, with
// six independent FFMA2 chains per lane.  Lanes 0-15 finish unit 2w, lanes 16-31 unit 2w+1.
// (template parameter KI: Hp = 128 KI; TRACE: clock64 phase stamps, diagnostic build)
template <int KI, bool TRACE>
__global__ void __launch_bounds__(256, 1) k_enc_recur2(EncDev e, int Tx) {
  pdl_wait();  // (no early trigger: the cooperative grid must not lose SMs to dependents)
  constexpr int Hp = 128 * KI, H4 = Hp / 4;
  __shared__ float4 h4buf[2][H4];  // by step parity: a warp reading step t never races the poll of t+1
  const int NB = e.NB, UPC = e.UPC, H = e.H;
  const int nthr = blockDim.x;
  const int dir = blockIdx.x / NB, cb = blockIdx.x % NB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ua = 2 * warp, ub = 2 * warp + 1;                 // the warp's units (CTA-local)
  const int side = lane >> 4;                                  // 0: lanes finish unit ua, 1: ub
  const int uloc = ua + side;
  const int jj = cb * UPC + uloc;                              // this lane's finishing unit (global)
  const bool unit = uloc < UPC && jj < H;
  long long* tr = (TRACE && blockIdx.x == 0 && threadIdx.x == 0) ? e.trace : nullptr;
  if (TRACE && tr) {
    tr[Tx * 8 + 0] = clock64();
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    tr[Tx * 8 + 5] = (long long)g;
  }
  const int C = 2 * H;
  const int per = (H + gridDim.x - 1) / gridDim.x;  // s0 outputs of this CTA (tail)
  extern __shared__ __align__(16) float wsm[];       // [per][C] rows of W_init^T (tail) | pin | ids
  __shared__ __align__(8) uint64_t wbar;             // completion of their bulk copy
  const int o_first = blockIdx.x * per, n_out = max(0, min(per, H - o_first));
  const bool bulk = (C % 4) == 0;
  if (bulk && threadIdx.x == 0) {
    mbar_init(&wbar, 1);
    fence_barrier_init();
    mbar_arrive_expect_tx(&wbar, (uint32_t)(n_out * C * 4));
    for (int r = 0; r < n_out; ++r)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(wsm + r * C)), "l"(e.W_initT + (int64_t)(o_first + r) * C), "r"(C * 4),
                   "r"(smem_u32(&wbar)) : "memory");
  }
  // weights: columns g * UPC + u of this CTA's [3 UPC][Hp] block (zero rows for u >= UPC)
  float4 wra[KI], wua[KI], wxa[KI], wrb[KI], wub[KI], wxb[KI];
  {
    const float4* src = reinterpret_cast<const float4*>(e.Uarr) + (size_t)(dir * NB + cb) * 3 * UPC * H4;
    const bool hb = ub < UPC;
#pragma unroll
    for (int i = 0; i < KI; ++i) {
      const int k = lane + 32 * i;
      wra[i] = src[(size_t)ua * H4 + k];
      wua[i] = src[(size_t)(UPC + ua) * H4 + k];
      wxa[i] = src[(size_t)(2 * UPC + ua) * H4 + k];
      wrb[i] = hb ? src[(size_t)ub * H4 + k] : make_float4(0.f, 0.f, 0.f, 0.f);
      wub[i] = hb ? src[(size_t)(UPC + ub) * H4 + k] : make_float4(0.f, 0.f, 0.f, 0.f);
      wxb[i] = hb ? src[(size_t)(2 * UPC + ub) * H4 + k] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  if (!bulk)
    for (int i = threadIdx.x; i < n_out * C; i += nthr) wsm[i] = __ldg(e.W_initT + (int64_t)o_first * C + i);
  unsigned* hx = e.hx + (size_t)dir * 2 * Hp;  // [2 parities][Hp] tagged words of this direction
  const int sdir = dir == 0 ? 1 : -1, s0 = dir == 0 ? 0 : Tx - 1;  // position of step t = s0 + sdir t
  // input projections of all steps (Tx <= kPinMax): ids, then 4-byte cp.async gathers
  const bool pre = Tx <= kPinMax;
  float* pin_s = wsm + per * C;                                          // [Tx][3][UPC]
  int* ids_s = reinterpret_cast<int*>(pin_s + (pre ? Tx * 3 * UPC : 0));  // [Tx]
  if (pre) {
    for (int t = threadIdx.x; t < Tx; t += nthr) {
      int id = __ldg(e.src + s0 + sdir * t);
      if (id < 0 || id >= e.Vs) {  // device-resident ids are validated here (nmt_ctx_check)
        atomicOr(e.err, ERR_TOKEN);
        id = 0;
      }
      ids_s[t] = id;
    }
    __syncthreads();
    const int per_t = 3 * UPC;
    for (int i = threadIdx.x; i < Tx * per_t; i += nthr) {
      const int t = i / per_t, g = (i % per_t) / UPC, u = i % UPC;
      const int uj = cb * UPC + u;
      if (uj < H)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(pin_s + i)),
                     "l"(e.encin + (int64_t)ids_s[t] * 6 * Hp + dir * 3 * Hp + g * Hp + uj) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
  }
  if (TRACE && tr)
    tr[Tx * 8 + 1] = clock64() + (long long)(wra[KI - 1].w == 12345.f) + (long long)(wxb[0].x == 12345.f);
  float hself = 0.f, hsum = 0.f;
  int npolls = 0;
  long long cyc_poll = 0, cyc_loop0 = TRACE ? clock64() : 0;
  for (int t = 0; t < Tx; ++t) {
    if (TRACE && tr) tr[t * 8 + 0] = clock64();
    const int j = s0 + sdir * t;
    float p_r = 0.f, p_u = 0.f, p_x = 0.f;
    if (unit) {
      if (pre) {
        const float* pt = pin_s + t * 3 * UPC + uloc;
        p_r = pt[0];
        p_u = pt[UPC];
        p_x = pt[2 * UPC];
      } else {
        int id = __ldg(e.src + j);
        if (id < 0 || id >= e.Vs) {
          if ((lane & 15) == 0) atomicOr(e.err, ERR_TOKEN);
          id = 0;
        }
        const float* pin = e.encin + (int64_t)id * 6 * Hp + dir * 3 * Hp + jj;
        p_r = __ldg(pin);
        p_u = __ldg(pin + Hp);
        p_x = __ldg(pin + 2 * Hp);
      }
    }
    if (TRACE && tr) tr[t * 8 + 1] = clock64();
    float2 ara = make_float2(0.f, 0.f), aua = ara, axa = ara, arb = ara, aub = ara, axb = ara;
    if (t > 0) {
      const unsigned tag = (unsigned)t & 3u;  // h_{t-1} was written with tag ((t-1)+1) mod 4
      float4* h4 = h4buf[t & 1];
      const unsigned* hsrc = hx + (size_t)(t & 1) * Hp;
      // <= 2 positions per thread (host-checked): both 256-bit loads are in flight before any wait
      const int k0 = threadIdx.x, k1 = threadIdx.x + nthr;
      const bool h0 = k0 < H4 && 4 * k0 < H, h1 = k1 < H4 && 4 * k1 < H;
      const unsigned need0 = (4 * k0 + 3 < H) ? 0xFu : ((1u << max(0, H - 4 * k0)) - 1u);  // real units only
      const unsigned need1 = (4 * k1 + 3 < H) ? 0xFu : ((1u << max(0, H - 4 * k1)) - 1u);
      unsigned a0 = 0, b0 = 0, c0 = 0, d0 = 0, a1 = 0, b1 = 0, c1 = 0, d1 = 0;
      if (h0)
        asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a0), "=r"(b0), "=r"(c0), "=r"(d0) : "l"(hsrc + 4 * k0) : "memory");
      if (h1)
        asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a1), "=r"(b1), "=r"(c1), "=r"(d1) : "l"(hsrc + 4 * k1) : "memory");
      auto settle = [&](bool has, int k, unsigned need, unsigned& a, unsigned& b, unsigned& c, unsigned& d) {
        if (!has) {
          if (k < H4) h4[k] = make_float4(0.f, 0.f, 0.f, 0.f);  // padded units (H < Hp) are never written
          return;
        }
        const long long tw = clock64();
        while (true) {
          ++npolls;
          const unsigned ok = ((a & 3u) == tag) | (((b & 3u) == tag) << 1) | (((c & 3u) == tag) << 2) |
                              (((d & 3u) == tag) << 3);
          if ((ok & need) == need) break;
          if (clock64() - tw > (1ll << 32)) asm volatile("trap;");  // watchdog (~2 s): fail, never hang
          asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(hsrc + 4 * k) : "memory");
        }
        h4[k] = make_float4((need & 1) ? __uint_as_float(a & ~3u) : 0.f, (need & 2) ? __uint_as_float(b & ~3u) : 0.f,
                            (need & 4) ? __uint_as_float(c & ~3u) : 0.f, (need & 8) ? __uint_as_float(d & ~3u) : 0.f);
      };
      settle(h0, k0, need0, a0, b0, c0, d0);
      settle(h1, k1, need1, a1, b1, c1, d1);
      if (TRACE && tr) tr[t * 8 + 2] = clock64();
      const long long cb0 = TRACE ? clock64() : 0;
      __syncthreads();  // (the only barrier of a step: buffer t&1 is rewritten at t+2, after t+1's barrier)
      if (TRACE && tr) tr[t * 8 + 3] = clock64();
      if (TRACE) cyc_poll += clock64() - cb0;
#pragma unroll
      for (int i = 0; i < KI; ++i) {
        const float4 h = h4[lane + 32 * i];
        const float2 hlo = make_float2(h.x, h.y), hhi = make_float2(h.z, h.w);
        ffma2(ara, make_float2(wra[i].x, wra[i].y), hlo);
        ffma2(aua, make_float2(wua[i].x, wua[i].y), hlo);
        ffma2(axa, make_float2(wxa[i].x, wxa[i].y), hlo);
        ffma2(arb, make_float2(wrb[i].x, wrb[i].y), hlo);
        ffma2(aub, make_float2(wub[i].x, wub[i].y), hlo);
        ffma2(axb, make_float2(wxb[i].x, wxb[i].y), hlo);
        ffma2(ara, make_float2(wra[i].z, wra[i].w), hhi);
        ffma2(aua, make_float2(wua[i].z, wua[i].w), hhi);
        ffma2(axa, make_float2(wxa[i].z, wxa[i].w), hhi);
        ffma2(arb, make_float2(wrb[i].z, wrb[i].w), hhi);
        ffma2(aub, make_float2(wub[i].z, wub[i].w), hhi);
        ffma2(axb, make_float2(wxb[i].z, wxb[i].w), hhi);
      }
    }
    // (h_0 = 0: the dot products are 0 at t = 0)
    float dra = ara.x + ara.y, dua = aua.x + aua.y, dxa = axa.x + axa.y;
    float drb = arb.x + arb.y, dub = aub.x + aub.y, dxb = axb.x + axb.y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {  // butterfly: every lane ends with all six sums
      dra += __shfl_xor_sync(0xffffffffu, dra, o);
      dua += __shfl_xor_sync(0xffffffffu, dua, o);
      dxa += __shfl_xor_sync(0xffffffffu, dxa, o);
      drb += __shfl_xor_sync(0xffffffffu, drb, o);
      dub += __shfl_xor_sync(0xffffffffu, dub, o);
      dxb += __shfl_xor_sync(0xffffffffu, dxb, o);
    }
    if (TRACE && tr) tr[t * 8 + 4] = clock64();
    if (unit) {
      const float dr = side ? drb : dra, du = side ? dub : dua, dx = side ? dxb : dxa;
      const float rg = sigmoid_fast(p_r + dr);
      const float ug = sigmoid_fast(p_u + du);
      const float ht = tanh_fast(rg * dx + p_x);
      hself = ug * hself + (1.f - ug) * ht;
      hsum += hself;
      const int cidx = dir * Hp + jj;  // padded context column
      const int role = lane & 15;
      if (role == 3) {  // publish h_t, tagged (t + 1) mod 4
        const unsigned word = (__float_as_uint(hself) & ~3u) | ((unsigned)(t + 1) & 3u);
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(hx + (size_t)((t + 1) & 1) * Hp + jj), "r"(word)
                     : "memory");
      } else if (role == 1) {
        e.ctx[(int64_t)j * 2 * Hp + cidx] = hself;
      } else if (role == 2) {
        __nv_bfloat16 hi, lo;
        split_bf16(hself, hi, lo);
        e.ctxbf[(int64_t)j * 4 * Hp + cidx] = hi;
        e.ctxbf[(int64_t)j * 4 * Hp + 2 * Hp + cidx] = lo;
      }
    }
    if (TRACE && tr) {
      tr[t * 8 + 5] = clock64();
      tr[t * 8 + 6] = npolls;
    }
  }
  // ---- E5: time means -> grid barrier -> s0 slices
  if (TRACE && tr) tr[Tx * 8 + 2] = clock64();
  if (TRACE && threadIdx.x == 0) {
    e.trace[(Tx + 1) * 8 + 2 * blockIdx.x] = clock64() - cyc_loop0;
    e.trace[(Tx + 1) * 8 + 2 * blockIdx.x + 1] = cyc_poll;
  }
  if (unit && (lane & 15) == 0) e.mean[dir * H + jj] = hsum / (float)Tx;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(e.bar) : "memory");
    int v;
    const long long t0 = clock64();
    do {
      asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(e.bar) : "memory");
      if (clock64() - t0 > (1ll << 32)) asm volatile("trap;");
    } while (v < (int)(e.epoch * gridDim.x));
  }
  __syncthreads();
  if (TRACE && tr) tr[Tx * 8 + 3] = clock64();
  if (unit && (lane & 15) == 3) {  // every CTA has read its last h: zero this unit's words for the next encode
    hx[jj] = 0u;
    hx[Hp + jj] = 0u;
  }
  // all 2H means at once (C <= 2Hp floats = the two h buffers), then a warp per s0 output
  float* msm = reinterpret_cast<float*>(h4buf);
  for (int k = threadIdx.x; k < C; k += nthr) msm[k] = __ldcg(e.mean + k);
  __syncthreads();
  const int nwarps = nthr >> 5;
  for (int w = warp; w < n_out; w += nwarps) {
    if (bulk) mbar_wait(&wbar, 0);
    const int o = o_first + w;
    const float* wrow = wsm + w * C;
    float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
    if (bulk) {
      for (int k = 4 * lane; k < C; k += 128) {
        const float4 mv = *reinterpret_cast<const float4*>(msm + k), wv = *reinterpret_cast<const float4*>(wrow + k);
        acc0 = fmaf(mv.x, wv.x, acc0);
        acc1 = fmaf(mv.y, wv.y, acc1);
        acc2 = fmaf(mv.z, wv.z, acc2);
        acc3 = fmaf(mv.w, wv.w, acc3);
      }
    } else {
      for (int k = lane; k < C; k += 32) acc0 = fmaf(msm[k], wrow[k], acc0);
    }
    float sacc = (acc0 + acc1) + (acc2 + acc3);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, off);
    if (lane == 0) e.S0[o] = tanhf(sacc + e.b_init[o]);
  }
  if (TRACE && tr) {
    tr[Tx * 8 + 4] = clock64();
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    tr[Tx * 8 + 6] = (long long)g;
  }
}

template <int KI, bool TRACE>
static void launch_recur2(const EncDev& e, int Tx, cudaStream_t st) {
  EncDev ee = e;
  void* args[] = {&ee, &Tx};
  const size_t smem = (size_t)((e.H + 2 * e.NB - 1) / (2 * e.NB)) * 2 * e.H * sizeof(float) +
                      (Tx <= kPinMax ? (size_t)Tx * (3 * e.UPC + 1) * sizeof(float) : 0);
  static std::atomic<size_t> attr[kMaxDevices];  // > 48 KB of dynamic shared memory needs the opt-in
  ensure_smem_attr(k_enc_recur2<KI, TRACE>, attr, smem);
  CK(cudaLaunchCooperativeKernel((void*)k_enc_recur2<KI, TRACE>, dim3(2 * e.NB), dim3(32 * ((e.UPC + 1) / 2)), args,
                                 smem, st));
  note_launch();
}

void enc_recur(const EncDev& e, int Tx, cudaStream_t st) {
  if (e.UPC > 16) throw NmtError(NMT_ERR_SHAPE, "encoder: UPC too large");
  if (2 * 32 * ((e.UPC + 1) / 2) < e.Hp / 4) throw NmtError(NMT_ERR_SHAPE, "encoder: > 2 polled words per thread");
  switch (e.Hp / 128) {
    case 1: e.trace ? launch_recur2<1, true>(e, Tx, st) : launch_recur2<1, false>(e, Tx, st); break;
    case 2: e.trace ? launch_recur2<2, true>(e, Tx, st) : launch_recur2<2, false>(e, Tx, st); break;
    case 3: e.trace ? launch_recur2<3, true>(e, Tx, st) : launch_recur2<3, false>(e, Tx, st); break;
    case 4: e.trace ? launch_recur2<4, true>(e, Tx, st) : launch_recur2<4, false>(e, Tx, st); break;
    case 5: e.trace ? launch_recur2<5, true>(e, Tx, st) : launch_recur2<5, false>(e, Tx, st); break;
    case 6: e.trace ? launch_recur2<6, true>(e, Tx, st) : launch_recur2<6, false>(e, Tx, st); break;
    case 7: e.trace ? launch_recur2<7, true>(e, Tx, st) : launch_recur2<7, false>(e, Tx, st); break;
    case 8: e.trace ? launch_recur2<8, true>(e, Tx, st) : launch_recur2<8, false>(e, Tx, st); break;
    default: throw NmtError(NMT_ERR_SHAPE, "encoder: dim_hid > 1024");
  }
}


// ===================================================================================== batched encoder
// nmt_encode_batch ("tensor-bound when B >~ 300 sentences are batched"): the
// recurrence of n sentences advances one time step per (GEMM, gate) pair.  Sentences are sorted by
// length (descending), so the rows still running at step t are a prefix [0, active(t)).
// GEMM of step t: [h_fwd | h_bwd] (bf16 hi|lo) . blockdiag([U|Ux]_fwd, [U|Ux]_bwd) -> G [n][6Hp];
// this kernel adds the precomputed input projections (EncIn[tok] = x.[W|Wx] + [b|bx]) and applies
// the DL4MT GRU: [r|u] = sigm(xW + b + hU); h~ = tanh(r*(hUx) + xWx + bx);
// h' = u*h + (1-u)*h~.  The forward direction reads token t, the backward token L_b - 1 - t, so each
// sentence's backward pass starts at its own last token (h_{Tx} = 0).
__global__ void k_encb_gates(EncBatchDev e, int t, int active) {
  pdl_enter();
  const int Hp = e.Hp, Cp = 2 * Hp, H4 = Hp / 4;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = idx / (2 * H4), rem = idx % (2 * H4), dir = rem / H4, j = (rem % H4) * 4;
  if (b >= active) return;
  const int o0 = e.tok_off[b], L = e.tok_off[b + 1] - o0;
  const int pos = dir ? L - 1 - t : t;
  const int tok = e.src[o0 + pos];
  const float* g = e.G + (int64_t)b * 6 * Hp + dir * 3 * Hp + j;
  const float* x = e.encin + (int64_t)tok * 6 * Hp + dir * 3 * Hp + j;
  const float4 gr = ld4_sum(g, e.ks, e.ps), gu = ld4_sum(g + Hp, e.ks, e.ps), gx = ld4_sum(g + 2 * Hp, e.ks, e.ps);
  const float4 xr = ld4(x), xu = ld4(x + Hp), xx = ld4(x + 2 * Hp);
  float* hp = e.h + (int64_t)b * Cp + dir * Hp + j;
  const float4 hv = ld4(hp);
  float4 o;
#define NMT_GRUE(c) { const float rg = sigm(xr.c + gr.c), ug = sigm(xu.c + gu.c); \
                      o.c = ug * hv.c + (1.f - ug) * tanhf(rg * gx.c + xx.c); }
  NMT_GRUE(x) NMT_GRUE(y) NMT_GRUE(z) NMT_GRUE(w)
#undef NMT_GRUE
  st4(hp, o);
  store_split4(e.A + (int64_t)b * 2 * Cp + dir * Hp + j, e.lo_a, o);
  st4(e.ctx[b] + (int64_t)pos * Cp + dir * Hp + j, o);
  store_split4(e.ctxbf + (int64_t)(o0 + pos) * 2 * Cp + dir * Hp + j, Cp, o);
}

// E5 input: mean_j ctx_j per sentence -> bf16 hi|lo operand of the s0 GEMM
__global__ void k_encb_mean(EncBatchDev e) {
  pdl_enter();
  const int Cp = 2 * e.Hp, b = blockIdx.y, k = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (k >= Cp) return;
  const int L = e.tok_off[b + 1] - e.tok_off[b];
  const float* c = e.ctx[b] + k;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int j = 0; j < L; ++j) {
    const float4 v = ld4(c + (int64_t)j * Cp);
    s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
  }
  const float inv = 1.f / (float)L;
  s.x *= inv; s.y *= inv; s.z *= inv; s.w *= inv;
  store_split4(e.Am + (int64_t)b * 2 * Cp + k, Cp, s);
}

// E6: s0 = tanh(mean ctx . W_init + b_init) into slot 0 of each sentence's state arena
__global__ void k_encb_s0(EncBatchDev e, const float* __restrict__ S0w, int ks, int64_t ps) {
  pdl_enter();
  const int b = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= e.Hp) return;
  float v = 0.f;
  if (j < e.H) v = tanhf(ld_sum(S0w + (int64_t)b * e.Hp + j, ks, ps) + e.b_init[j]);
  e.S0[b][j] = v;
}

// E7 output: pctx rows of the token-major batch GEMM (+ b_att) scattered to each sentence's pctx
__global__ void k_encb_pctx(EncBatchDev e, const float* __restrict__ P, int ks, int64_t ps, int n_tok) {
  pdl_enter();
  const int Cp = 2 * e.Hp, C4 = Cp / 4;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int r = (int)(idx / C4), k = (int)(idx % C4) * 4;
  if (r >= n_tok) return;
  const int b = e.row_b[r], pos = r - e.tok_off[b];
  float4 v = ld4_sum(P + (int64_t)r * Cp + k, ks, ps);
  const float4 bb = ld4(e.b_att + k);
  v.x += bb.x; v.y += bb.y; v.z += bb.z; v.w += bb.w;
  st4(e.pctx[b] + (int64_t)pos * Cp + k, v);
  bool b0, b1, b2, b3;
  const float4 ev = make_float4(exp2x_clamped(v.x, b0), exp2x_clamped(v.y, b1), exp2x_clamped(v.z, b2),
                                exp2x_clamped(v.w, b3));
  st4(e.epctx[b] + (int64_t)pos * Cp + k, ev);
  if (b0 | b1 | b2 | b3) atomicOr(e.cnt[b] + CNT_BIGP, 1);
}

// context (re)initialisation of n arenas in one launch (k_ctx_reset per blockIdx.y)
__global__ void k_ctx_reset_many(const CtxDev* __restrict__ cs, const int64_t* __restrict__ hcaps) {
  pdl_enter();
  const CtxDev c = cs[blockIdx.y];
  const int64_t hcap = hcaps[blockIdx.y];
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = i0; i < hcap; i += (int64_t)gridDim.x * blockDim.x) {
    c.hkeys[i] = ~0ull;
    c.hvals[i] = INT32_MIN;
  }
  if (i0 == 0) {
    c.counters[CNT_NODES] = 1;
    c.counters[CNT_SLOTS] = 2;
    c.counters[CNT_ERR] = 0;
    c.counters[CNT_R] = 0;
    c.counters[CNT_BIGP] = 0;
    c.node_word[0] = -1;
    c.node_parent[0] = -1;
    c.node_src[0] = 0;
    c.node_slot[0] = -1;
  }
}

void encb_gates(const EncBatchDev& e, int t, int active, cudaStream_t st) {
  const int64_t n = (int64_t)active * 2 * (e.Hp / 4);
  launch_pdl(k_encb_gates, (unsigned)((n + 255) / 256), 256, 0, st, e, t, active);
  CK_LAUNCH();
}
void encb_mean(const EncBatchDev& e, cudaStream_t st) {
  launch_pdl(k_encb_mean, dim3((2 * e.Hp / 4 + 127) / 128, e.n), 128, 0, st, e);
  CK_LAUNCH();
}
void encb_s0(const EncBatchDev& e, const float* S0w, int ks, int64_t ps, cudaStream_t st) {
  launch_pdl(k_encb_s0, dim3((e.Hp + 127) / 128, e.n), 128, 0, st, e, S0w, ks, ps);
  CK_LAUNCH();
}
void encb_pctx(const EncBatchDev& e, const float* P, int ks, int64_t ps, int n_tok, cudaStream_t st) {
  const int64_t n = (int64_t)n_tok * (2 * e.Hp / 4);
  launch_pdl(k_encb_pctx, (unsigned)((n + 255) / 256), 256, 0, st, e, P, ks, ps, n_tok);
  CK_LAUNCH();
}
void ctx_reset_many(const CtxDev* cs, const int64_t* hcaps, int n, int64_t hcap_max, cudaStream_t st) {
  const int64_t b = std::min<int64_t>((hcap_max + 255) / 256, 64);
  launch_pdl(k_ctx_reset_many, dim3((unsigned)std::max<int64_t>(b, 1), n), 256, 0, st, cs, hcaps);
  CK_LAUNCH();
}

}  // namespace nmt
