// gemm.cu - persistent warp-specialised tcgen05 GEMM engine for sm_100a.
//
//   C[M x N] = A[M x K] . B[N x K]^T        A, B bf16 K-major in HBM, fp32 accumulate in TMEM.
//
// Roles (192 threads, 1 CTA / SM): warp 0 = TMA producer (one elected lane), warp 1 = TMEM
// allocator + MMA issuer (one elected lane), warps 2..5 = epilogue (thread = accumulator row =
// TMEM lane).  Operand tiles 128 x 64 (A) and BN x 64 (B) are staged by TMA into a STAGES-deep
// 128B-swizzled ring guarded by full/empty mbarriers; accumulators are double buffered in TMEM
// (2 x BN fp32 columns) so the epilogue of tile i overlaps the MMAs of tile i+1.
//
// Split precision (NMT_PREC_FP32CLASS): x = hi + lo (both bf16); A.B ~ Ahi.Bhi + Ahi.Blo + Alo.Bhi,
// realised as three K passes over the same accumulator; the lo halves live at a column offset
// of the same tensors (a_lo_off / b_lo_off).
// K ranges per N range ("regions") let one GEMM compute [gates | hUx | cWcx] of a GRU over a
// concatenated activation buffer without multiplying zero blocks.
//
// Epilogues: EPI_STORE writes fp32 (+bias[col]); EPI_LSE is the fused vocabulary epilogue of
// step D8: per (row, N-tile) running max, sum of exp and argmax of the logits -
// the logits never leave the chip (PAPER.md:120 computes P_i explicitly; we never do).
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <vector>
#include <mutex>
#include <tuple>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "internal.h"
#include "kernels.h"

namespace nmt {

constexpr int BM = 128, BK = 64;
constexpr int EPI_STORE = 0, EPI_LSE = 1, EPI_TOPK = 2;  // TOPK: runs like LSE, keeps the kTopK best logits
constexpr int EPI_GRU = 3;  // fused GRU gates (one tile per item like EPI_STORE, no split-K)
// fused decoder GRU2 (D6): per 32-unit group the B rows are [hx | r | u | cx]; the s1 K range multiplies
// rows hx, r, u (MMA N = 192 over the first 96 rows of each CTA's half) into accumulator D1, the c K range
// rows r, u, cx (N = 192 from row 32) into D2, so no zero block is multiplied; single-buffered TMEM
constexpr int EPI_GRU2 = 4;
// fused readout (D7) on 256 x 128 CTA-pair tiles: each epilogue warp's 64 columns give 32 maxout (or 64
// tanh) outputs of its row
constexpr int EPI_READOUT = 5;
template <int EPI>
constexpr bool single_acc() { return EPI == EPI_GRU2; }
constexpr int EPI_WARPS = 8;  // 2 per TMEM lane quadrant, each owning half of the tile's columns
constexpr int GEMM_THREADS = 64 + 32 * EPI_WARPS;

constexpr int kAresKB = 8;  // ARES: k-blocks of the resident A tile (K <= 512: the vocabulary GEMM's Ep)

// PAIR (cta_group::2): a cluster of 2 CTAs computes 256 x BN tiles - M = 256 across the pair, each
// CTA holds its 128 rows of A and HALF of the B tile, so per SM a k-block moves (16 + BN/8) KB for
// the MMA work of a 128 x BN tile.  Protocol (as CUTLASS' 2SM kernels): both CTAs TMA into their own
// smem and count bytes on the leader's full barrier (+1 remote arrive from the peer); the leader
// issues the MMAs and commits with multicast to both CTAs' empty / tfull barriers; every epilogue
// warp of both CTAs arrives on the leader's tempty barrier.
template <int BN, int STAGES, int EPI, bool PAIR, bool ARES = false>
struct GemmSmem {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_ROWS = PAIR ? BN / 2 : BN;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  // EPI_STORE: per epilogue warp two 32 x 32 fp32 staging tiles (128B-swizzled) for TMA stores
  static constexpr int C_BYTES = EPI == 0 ? EPI_WARPS * 2 * 4096 : 0;
  // ARES (A resident): the A tile of a work item's m-tile, all its k-blocks (K <= kAresKB * 64), stays in
  // shared memory for the item's whole n-run; the stage ring carries only B
  static constexpr int A_RING = ARES ? 0 : A_BYTES;
  static constexpr int A_RES = ARES ? kAresKB * A_BYTES : 0;
  static constexpr int BYTES = 1024 + A_RES + STAGES * (A_RING + B_BYTES) + C_BYTES + (2 * STAGES + 6) * 8 + 16;
};

struct RegionK {
  int k0, k1;  // in units of BK blocks
  int ks;      // split-K factor of the region
};

struct TileCoord {
  int m, n, s;
};
NMT_DEV TileCoord tile_of(int t, int num_m, int num_n) {
  return TileCoord{t % num_m, (t / num_m) % num_n, t / (num_m * num_n)};
}
// Work items over m-tiles of CM = 128 (or 256 rows for a CTA pair) and n-tiles of BN:
// EPI_STORE -> one tile per item (m fastest, so concurrent units share B tiles in L2).
// EPI_LSE -> item = (m-tile, contiguous run of n-tiles): the unit keeps each row's running
// (max, sum, argmax) across its run and emits ONE partial per row and run half.
struct Item {
  int m, s, n0, n1, c;
};
// EPI_STORE items go region by region; inside a region m is fastest, then n, then the K split.
struct Sched {
  int num_m, num_n, cpm, chunk, items;
  int nreg, nt_end[4], ks[4], it_end[4];  // per region: n-tile end, split count, cumulative items
  NMT_DEV Item item(int i) const {
    if (cpm == 0) {
      int r = 0, nt0 = 0, i0 = 0;
#pragma unroll 1
      while (r < nreg - 1 && i >= it_end[r]) {
        nt0 = nt_end[r];
        i0 = it_end[r];
        ++r;
      }
      const int li = i - i0, ntr = nt_end[r] - nt0;
      const int rest = li / num_m, n = nt0 + rest % ntr;
      return Item{li % num_m, rest / ntr, n, n + 1, 0};
    }
    const int m = i / cpm, c = i % cpm;
    const int n0 = min(num_n, c * chunk);
    return Item{m, 0, n0, min(num_n, n0 + chunk), c};
  }
};
template <int EPI>
NMT_DEV Sched make_sched(const GemmShape& g, int M, int CM, int BN, int units) {
  Sched s;
  s.num_m = (M + CM - 1) / CM;
  s.num_n = g.N / BN;
  s.nreg = g.nreg;
  if (EPI == EPI_LSE || EPI == EPI_TOPK) {  // (m-tile, n-run) items
    s.cpm = max(1, units / max(1, s.num_m));
    s.chunk = (s.num_n + s.cpm - 1) / s.cpm;
    s.items = s.num_m * s.cpm;
  } else {
    s.cpm = 0;
    s.chunk = 1;
    int nt0 = 0, acc = 0;
    for (int r = 0; r < g.nreg; ++r) {
      const int nt1 = r < g.nreg - 1 ? g.reg_n_end[r] / BN : s.num_n;
      s.ks[r] = g.reg_ks[r] > 0 ? g.reg_ks[r] : g.ksplit;
      acc += s.num_m * (nt1 - nt0) * s.ks[r];
      s.nt_end[r] = nt1;
      s.it_end[r] = acc;
      nt0 = nt1;
    }
    s.items = acc;
  }
  return s;
}

NMT_DEV RegionK region_of(const GemmShape& g, int n0) {
  int r = 0;
#pragma unroll 1
  while (r < g.nreg - 1 && n0 >= g.reg_n_end[r]) ++r;
  return RegionK{g.reg_k0[r] / BK, g.reg_k1[r] / BK, g.reg_ks[r] > 0 ? g.reg_ks[r] : g.ksplit};
}

// GRU gate math of the fused epilogues on the SFU: ex2.approx + rcp.approx based, |err| ~ 1e-7 (the
// IEEE expf / division / tanhf versions made these epilogues issue-bound: ~7 us per tile on 8 warps)
NMT_DEV float gru_sigm(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
NMT_DEV float gru_tanh(float x) { return 1.f - __fdividef(2.f, 1.f + __expf(2.f * x)); }
NMT_DEV uint32_t gru_pk(float lo, float hi) {
  uint32_t y;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(hi), "f"(lo));
  return y;
}
// 4 values as bf16 (and the bf16 residuals at +lo_off when lo_off > 0)
NMT_DEV void gru_store4(__nv_bfloat16* p, int lo_off, float a, float b, float c, float d) {
  const uint32_t h01 = gru_pk(a, b), h23 = gru_pk(c, d);
  *reinterpret_cast<uint2*>(p) = make_uint2(h01, h23);
  if (lo_off > 0)
    *reinterpret_cast<uint2*>(p + lo_off) =
        make_uint2(gru_pk(a - __uint_as_float(h01 << 16), b - __uint_as_float(h01 & 0xffff0000u)),
                   gru_pk(c - __uint_as_float(h23 << 16), d - __uint_as_float(h23 & 0xffff0000u)));
}

// diagnostic phase stamps (NMT_DIAG builds with NMT_GEMM_TRACE): entry, prologue done, inputs ready,
// first stage landed (MMA), last MMA issued, first accumulator ready (epilogue), epilogue done, exit
#ifdef NMT_DIAG
#define GTRACE(ev)                                                                              \
  do {                                                                                          \
    if (ep.trace) {                                                                             \
      unsigned long long t_;                                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                    \
      ep.trace[blockIdx.x * 8 + (ev)] = t_;                                                     \
    }                                                                                           \
  } while (0)
#else
#define GTRACE(ev) \
  do {             \
  } while (0)
#endif

// Per-CTA view of the engine's shared memory, barriers and TMEM, and the roles' pipeline positions
// (a role function called twice in one launch would continue the same stage ring).
template <int BN, int STAGES, int EPI, bool PAIR, bool ARES = false>
struct GemmCta {
  using S = GemmSmem<BN, STAGES, EPI, PAIR, ARES>;
  static constexpr int CM = PAIR ? 2 * BM : BM;  // rows of a tile (per CTA pair)
  uint8_t *sA, *sB, *sC;
  uint64_t *full, *empty, *tfull, *tempty;
  uint64_t *afull, *aempty;  // ARES: resident A tile landed / released by the MMAs of its item
  uint32_t* tmem_slot;
  uint32_t tmem;
  int warp, lane;
  uint32_t rank;
  bool leader;
  int unit, nunits;
  // pipeline positions (each used by one role)
  int p_stage = 0, m_stage = 0, m_it = 0, e_it = 0, p_item = 0, m_item = 0;
  uint32_t p_phase = 0, m_phase = 0;

  NMT_DEV void carve(uint8_t* smem_raw) {
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    sA = smem;  // ARES: the resident A tile [kAresKB][A_BYTES]; else the A halves of the stage ring
    sB = smem + S::A_RES + STAGES * S::A_RING;
    sC = sB + STAGES * S::B_BYTES;  // (1024-aligned: A/B stage sizes are multiples of 1 KB)
    full = reinterpret_cast<uint64_t*>(sC + S::C_BYTES);
    empty = full + STAGES;
    tfull = empty + STAGES;
    tempty = tfull + 2;
    afull = tempty + 2;
    aempty = afull + 1;
    tmem_slot = reinterpret_cast<uint32_t*>(aempty + 1);
    warp = threadIdx.x >> 5;
    lane = threadIdx.x & 31;
    rank = PAIR ? cluster_ctarank() : 0;
    leader = rank == 0;
    unit = PAIR ? blockIdx.x / 2 : blockIdx.x;
    nunits = PAIR ? gridDim.x / 2 : gridDim.x;
  }
  // barrier init (warp 0) and TMEM allocation (warp 1), then a CTA / cluster barrier
  NMT_DEV void setup() {
    if (warp == 0 && lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full[s], PAIR ? 2 : 1);  // (pair: the leader's expect_tx arrive + the peer's remote arrive)
        mbar_init(&empty[s], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&tfull[a], 1);
        mbar_init(&tempty[a], (PAIR ? 2 : 1) * EPI_WARPS);
      }
      mbar_init(afull, PAIR ? 2 : 1);
      mbar_init(aempty, 1);
      fence_barrier_init();
    }
    if (warp == 1) {
      if constexpr (PAIR) tmem_alloc_pair(tmem_slot, 2 * BN);
      else tmem_alloc(tmem_slot, 2 * BN);
    }
    tc_fence_before();
    if constexpr (PAIR) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    tmem = *tmem_slot;
  }
  NMT_DEV void teardown() {
    __syncthreads();
    if constexpr (PAIR) cluster_sync();
    if (warp == 1) {
      tc_fence_after();
      if constexpr (PAIR) tmem_dealloc_pair(tmem, 2 * BN);
      else tmem_dealloc(tmem, 2 * BN);
    }
  }
};

// ---- TMA producer: the whole warp 0 runs the (warp-uniform) loop, one elected lane issues (both CTAs of a
// pair load their halves)
template <int BN, int STAGES, int EPI, bool PAIR, bool ARES = false>
NMT_DEV void gemm_produce(GemmCta<BN, STAGES, EPI, PAIR, ARES>& cx, const CUtensorMap* tmA, const CUtensorMap* tmB,
                          const CUtensorMap* tmB2, const GemmShape& g, const Sched& sc) {
  using S = GemmSmem<BN, STAGES, EPI, PAIR, ARES>;
  constexpr int CM = GemmCta<BN, STAGES, EPI, PAIR, ARES>::CM;
  const uint32_t full0 = PAIR ? mapa_shared(smem_u32(cx.full), 0) : 0;
  for (int w = cx.unit; w < sc.items; w += cx.nunits) {
    const Item itm = sc.item(w);
    if constexpr (ARES) {  // the item's A tile once: all k-blocks (single pass, one region, no split)
      const RegionK rk = region_of(g, itm.n0 * BN);
      const int nkb = rk.k1 - rk.k0;
      if (cx.p_item > 0) mbar_wait(cx.aempty, (cx.p_item - 1) & 1);  // the previous item's MMAs are done with A
      const int arow = itm.m * CM + cx.rank * BM;
      if (elect_one()) {
        if constexpr (PAIR) {
          if (cx.leader) mbar_arrive_expect_tx(cx.afull, 2 * nkb * S::A_BYTES);
          else mbar_arrive_cluster(mapa_shared(smem_u32(cx.afull), 0));
          for (int kb = 0; kb < nkb; ++kb)
            tma_load_2d_pair(tmA, cx.afull, cx.sA + kb * S::A_BYTES, g.a_col0 + (rk.k0 + kb) * BK, arow);
        } else {
          mbar_arrive_expect_tx(cx.afull, nkb * S::A_BYTES);
          for (int kb = 0; kb < nkb; ++kb)
            tma_load_2d(tmA, cx.afull, cx.sA + kb * S::A_BYTES, g.a_col0 + (rk.k0 + kb) * BK, arow);
        }
      }
      __syncwarp();
      ++cx.p_item;
    }
    for (int n = itm.n0; n < itm.n1; ++n) {
      const TileCoord tc{itm.m, n, itm.s};
      const RegionK rk = region_of(g, tc.n * BN);
      const int nkbp = rk.k1 - rk.k0, nkb = g.passes * nkbp;
      const int chunk = (nkb + rk.ks - 1) / rk.ks;
      const int i1 = min(nkb, (tc.s + 1) * chunk);
      for (int i = tc.s * chunk; i < i1; ++i) {
        const int pass = i / nkbp, kb = rk.k0 + i % nkbp;
        const int aoff = g.a_col0 + (pass == 2 ? g.a_lo_off : 0);
        const int boff = (pass == 1 ? g.b_lo_off : 0);
        const int stage = cx.p_stage;
        mbar_wait(&cx.empty[stage], cx.p_phase ^ 1);
        const int arow = tc.m * CM + cx.rank * BM, brow = tc.n * BN + cx.rank * S::B_ROWS + g.n_off;
        const bool in_b2 = kb >= g.b2_kb0 && kb < g.b2_kb1;  // (second B operand: never with B panels)
        const int kj = (g.b2_kb1 > 0 && kb >= g.b2_kb1) ? g.kjump : 0;
        const int bx = in_b2 ? (pass == 1 ? g.b2_lo_off : 0) + (kb - g.b2_kb0) * BK
                             : (g.b_panel_rows ? 0 : boff + kb * BK + kj);
        const int by = (!in_b2 && g.b_panel_rows) ? (boff / BK + kb) * g.b_panel_rows + brow : brow;
        const CUtensorMap* tb = in_b2 ? tmB2 : tmB;
        if (elect_one()) {
          if constexpr (PAIR) {
            if (cx.leader) mbar_arrive_expect_tx(&cx.full[stage], 2 * (S::A_RING + S::B_BYTES));
            else mbar_arrive_cluster(full0 + stage * 8);
            if constexpr (!ARES)
              tma_load_2d_pair(tmA, &cx.full[stage], cx.sA + stage * S::A_BYTES, aoff + kb * BK + kj, arow);
            tma_load_2d_pair(tb, &cx.full[stage], cx.sB + stage * S::B_BYTES, bx, by);
          } else {
            mbar_arrive_expect_tx(&cx.full[stage], S::A_RING + S::B_BYTES);
            if constexpr (!ARES)
              tma_load_2d(tmA, &cx.full[stage], cx.sA + stage * S::A_BYTES, aoff + kb * BK + kj, arow);
            tma_load_2d(tb, &cx.full[stage], cx.sB + stage * S::B_BYTES, bx, by);
          }
        }
        __syncwarp();
        if (++cx.p_stage == STAGES) {
          cx.p_stage = 0;
          cx.p_phase ^= 1;
        }
      }
    }
  }
}

// ---- MMA issuer: the whole warp 1 of the pair's leader runs the (warp-uniform) loop, so descriptors and
// TMEM addresses live in uniform registers; one elected lane issues a k-block's MMAs and its commit
// (lane-divergent issue cost ~20 instructions per MMA in ELECT / R2UR broadcast loops)
template <int BN, int STAGES, int EPI, bool PAIR, bool ARES = false>
NMT_DEV void gemm_mma(GemmCta<BN, STAGES, EPI, PAIR, ARES>& cx, const GemmShape& g, const Sched& sc, const EpiParams& ep) {
  using S = GemmSmem<BN, STAGES, EPI, PAIR, ARES>;
  constexpr int CM = GemmCta<BN, STAGES, EPI, PAIR, ARES>::CM;
  constexpr uint32_t idesc = idesc_bf16(CM, BN);
  constexpr uint32_t idesc2 = idesc_bf16(CM, 192);  // (EPI_GRU2, EPI_GRU)
  const uint64_t adesc0 = sdesc_sw128(smem_u32(cx.sA)), bdesc0 = sdesc_sw128(smem_u32(cx.sB));
  for (int w = cx.unit; w < sc.items; w += cx.nunits) {
    const Item itm = sc.item(w);
    if constexpr (ARES) {
      mbar_wait(cx.afull, cx.m_item & 1);  // the item's resident A tile
      tc_fence_after();
    }
    for (int n = itm.n0; n < itm.n1; ++n, ++cx.m_it) {
      const TileCoord tc{itm.m, n, itm.s};
      const RegionK rk = region_of(g, tc.n * BN);
      const int acc = single_acc<EPI>() ? 0 : cx.m_it & 1;
      const uint32_t aph = single_acc<EPI>() ? cx.m_it & 1 : (cx.m_it >> 1) & 1;
      mbar_wait(&cx.tempty[acc], aph ^ 1);
      tc_fence_after();
      const uint32_t d = cx.tmem + acc * BN;
      const int nkb_s1 = ep.Hp / BK;  // (EPI_GRU2: k-blocks of the s1 range)
      const int nkb_all = g.passes * (rk.k1 - rk.k0);
      const int chunk = (nkb_all + rk.ks - 1) / rk.ks;
      const int nkb = min(nkb_all, (tc.s + 1) * chunk) - tc.s * chunk;
      for (int i = 0; i < nkb; ++i) {
        const int stage = cx.m_stage;
        mbar_wait(&cx.full[stage], cx.m_phase);
        tc_fence_after();
        if (cx.lane == 0 && cx.m_it == 0 && i == 0) GTRACE(3);
        // descriptor start-address field: (smem address >> 4), +2 per 32 bytes (16 bf16 of K)
        const uint64_t ad = adesc0 + (uint64_t)((ARES ? i : stage) * (S::A_BYTES >> 4));  // (ARES: k-block i)
        const uint64_t bd = bdesc0 + (uint64_t)(stage * (S::B_BYTES >> 4));
        if (elect_one()) {
          if constexpr (EPI == EPI_GRU2) {
            static_assert(PAIR && BN == 256, "EPI_GRU2: CTA pairs, 2 groups per tile");
            const int kbp = i % (rk.k1 - rk.k0);        // k-block within the pass
            const bool c_rng = kbp >= nkb_s1;
            const int first = c_rng ? nkb_s1 : 0;       // first k-block of this accumulator's range
            const uint32_t dd = d + (c_rng ? 192 : 0);  // D2 follows D1 (384 of the 512 columns)
            const uint64_t bo = c_rng ? (32 * 128) >> 4 : 0;  // rows r, u, cx start 32 rows into the half
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) mma_bf16_pair(dd, ad + 2 * k, bd + bo + 2 * k, idesc2, (i != first || k != 0));
          } else {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              // (EPI_GRU: N = 192, the first 96 B rows [r | u | x] of each CTA's group; the zero quarter is skipped)
              if constexpr (PAIR) mma_bf16_pair(d, ad + 2 * k, bd + 2 * k, EPI == EPI_GRU ? idesc2 : idesc, (i | k) != 0);
              else mma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (i | k) != 0);
            }
          }
          if constexpr (PAIR) mma_commit_pair(&cx.empty[stage]);
          else mma_commit(&cx.empty[stage]);
        }
        __syncwarp();
        if (++cx.m_stage == STAGES) {
          cx.m_stage = 0;
          cx.m_phase ^= 1;
        }
      }
      if (elect_one()) {
        if constexpr (PAIR) mma_commit_pair(&cx.tfull[acc]);
        else mma_commit(&cx.tfull[acc]);
      }
      __syncwarp();
    }
    if constexpr (ARES) {  // the item's MMAs done: both CTAs' producers may reload A
      if (elect_one()) {
        if constexpr (PAIR) mma_commit_pair(cx.aempty);
        else mma_commit(cx.aempty);
      }
      __syncwarp();
      ++cx.m_item;
    }
  }
  if (cx.lane == 0) GTRACE(4);
}

// ---- epilogue warps 2..9 (each CTA: its 128 rows of the tile)
template <int BN, int STAGES, int EPI, bool PAIR, bool ARES = false>
NMT_DEV void gemm_epilogue(GemmCta<BN, STAGES, EPI, PAIR, ARES>& cx, const CUtensorMap* tmC, const GemmShape& g, int M,
                           const Sched& sc, const EpiParams& ep) {
  constexpr int CM = GemmCta<BN, STAGES, EPI, PAIR, ARES>::CM;
  const int warp = cx.warp, lane = cx.lane;
  const uint32_t rank = cx.rank, tmem = cx.tmem;
  const bool leader = cx.leader;
  uint64_t* tfull = cx.tfull;
  uint64_t* tempty = cx.tempty;
  uint8_t* sC = cx.sC;
  const int q = warp & 3;               // TMEM lane quadrant accessible to this warp
  const int half = (warp - 2) >> 2;     // which half of the tile's columns
  constexpr int COLS = BN / 2;
  const int row_in_tile = q * 32 + lane;
  const uint32_t tempty0 = PAIR ? mapa_shared(smem_u32(tempty), 0) : 0;
  int& it = cx.e_it;
  for (int w = cx.unit; w < sc.items; w += cx.nunits) {
    const Item itm = sc.item(w);
    const int grow = itm.m * CM + rank * BM + row_in_tile;
    const bool valid = grow < M;
    constexpr float LOG2E = 1.4426950408889634f;
    float mx = -INFINITY, s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;  // LSE running state (per run)
    int am = 0;
    float tv[EPI == EPI_TOPK ? kTopK : 1];  // TOPK: best logits of the run, descending (ties: lower column)
    int ti[EPI == EPI_TOPK ? kTopK : 1];
    if constexpr (EPI == EPI_TOPK) {
#pragma unroll
      for (int q = 0; q < kTopK; ++q) {
        tv[q] = -INFINITY;
        ti[q] = INT32_MAX;
      }
    }
    for (int n = itm.n0; n < itm.n1; ++n, ++it) {
      const int acc = single_acc<EPI>() ? 0 : it & 1;
      const uint32_t aph = single_acc<EPI>() ? it & 1 : (it >> 1) & 1;
      const int colbase = n * BN + half * COLS;
      // EPI_GRU: this warp's COLS = 128 columns are one 32-unit group [r | u | h~ | pad] of its row, done
      // in 4 chunks of 8 units.  The gx (r, u, x) and previous-state values arrive as 256-bit loads (full
      // 32-byte sectors), all issued before the accumulator wait, so their latency hides under the main loop.
      float gin[EPI == EPI_GRU ? 4 : 1][4][8];
      const float* gxr = nullptr;
      const float* sp = nullptr;
      auto gru_fetch = [&](int c, float(&b)[4][8]) {
        if (!valid) return;
        ld8_nc(gxr + 8 * c, b[0]);
        ld8_nc(gxr + ep.Hp + 8 * c, b[1]);
        ld8_nc(gxr + 2 * ep.Hp + 8 * c, b[2]);
        ld8(sp + 8 * c, b[3]);
      };
      if constexpr (EPI == EPI_GRU) {
        if (valid) {
          const int j0 = (colbase >> 7) * 32;
          const int y = ep.row_y[grow];
          gxr = ep.gx + (int64_t)(y < 0 ? ep.y_bos : y) * ep.gx_ld + j0;
          sp = ep.S + (int64_t)ep.row_src[grow] * ep.Hp + j0;
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) gru_fetch(c, gin[c]);  // all four chunks in flight under the main loop
      }
      float s1in[EPI == EPI_GRU2 ? 4 : 1][8];  // EPI_GRU2: the row's s1 for the group's 32 units
      float bia[EPI == EPI_GRU2 ? 2 : 1][3][8];  // EPI_GRU2: b_nl (r, u) and bx_nl, two chunks ahead
      float epj[EPI == EPI_READOUT ? COLS / 8 : 1][8];  // EPI_READOUT: Eproj[y] at the warp's columns
      if constexpr (EPI == EPI_READOUT) {
        if (valid) {
          const int dst = ep.row_dst[grow];
          const int y = dst >= 0 ? ep.row_y[grow] : -1;
          const float* epr = ep.Eproj + (int64_t)(y < 0 ? ep.V : y) * ep.ldc + colbase;
#pragma unroll
          for (int c = 0; c < COLS / 8; ++c) ld8_nc(epr + 8 * c, epj[c]);
        }
      }
      auto bias_fetch = [&](int c, float(&b)[3][8]) {
        const int jb = (colbase >> 7) * 32 + 8 * c;
        ld8_nc(ep.b_nl + jb, b[0]);
        ld8_nc(ep.b_nl + ep.Hp + jb, b[1]);
        ld8_nc(ep.bx_nl + jb, b[2]);
      };
      if constexpr (EPI == EPI_GRU2) {
        if (valid) {
          const float* s1p = ep.S1 + (int64_t)grow * ep.Hp + (colbase >> 7) * 32;
#pragma unroll
          for (int c = 0; c < 4; ++c) ld8(s1p + 8 * c, s1in[c]);
        }
        bias_fetch(0, bia[0]);
        bias_fetch(1, bia[1]);
      }
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      if (it == 0 && warp == 2 && lane == 0) GTRACE(5);
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * BN + half * (EPI == EPI_GRU ? 96 : COLS);
      if constexpr (EPI == EPI_STORE) {
        // TMEM -> registers (+bias) -> 128B-swizzled 32x32 smem tile -> TMA store (coalesced)
        uint8_t* stile = sC + (size_t)(warp - 2) * 2 * 4096;
        const int row0 = itm.s * ep.rows_per_split + itm.m * CM + rank * BM + q * 32;
#pragma unroll 1
        for (int c = 0; c < COLS; c += 32) {
          uint8_t* buf = stile + ((c >> 5) & 1) * 4096;
          if (lane == 0) bulk_wait_read<1>();  // the store that used this buffer has read it
          __syncwarp();
          float v[32];
          tmem_ld32_nowait(tbase + c, v);
          tmem_wait_ld_dep(v);
          if (ep.bias) {
            const float4* b = reinterpret_cast<const float4*>(ep.bias + colbase + c);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 bb = __ldg(b + j);
              v[4 * j] += bb.x; v[4 * j + 1] += bb.y; v[4 * j + 2] += bb.z; v[4 * j + 3] += bb.w;
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4* dst = reinterpret_cast<float4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4));
            *dst = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(tmC, buf, colbase + c, row0);
            bulk_commit();
          }
        }
      } else if constexpr (EPI == EPI_TOPK) {  // running top-kTopK of this warp's COLS logits of the row
#pragma unroll 1
        for (int c = 0; c < COLS; c += 32) {
          float v[32];
          tmem_ld32_nowait(tbase + c, v);
          tmem_wait_ld_dep(v);
          const int col0 = colbase + c + g.n_off;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (v[j] > tv[kTopK - 1] && col0 + j < ep.n_valid) {  // (rare once the list is full)
              float x = v[j];
              int xi = col0 + j;
#pragma unroll
              for (int q = 0; q < kTopK; ++q) {  // sorted insert; an equal value stays behind
                if (x > tv[q]) {
                  const float tx = tv[q];
                  const int txi = ti[q];
                  tv[q] = x;
                  ti[q] = xi;
                  x = tx;
                  xi = txi;
                }
              }
            }
          }
        }
      } else if constexpr (EPI == EPI_GRU) {
        static_assert(BN / 2 == 128, "EPI_GRU: one 32-unit group per epilogue warp");
        const int j0 = (colbase >> 7) * 32;
        float* s1 = ep.S1 + (int64_t)grow * ep.Hp + j0;
        __nv_bfloat16* xo = ep.X + (int64_t)grow * ep.ldx + j0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float vr[8], vu[8], vx[8];
          tmem_ld8_nowait(tbase + 8 * c, vr);
          tmem_ld8_nowait(tbase + 32 + 8 * c, vu);
          tmem_ld8_nowait(tbase + 64 + 8 * c, vx);
          tmem_wait_ld();
          reg_dep8(vr);
          reg_dep8(vu);
          reg_dep8(vx);
          float(&b)[4][8] = gin[c];
          float o[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float rg = gru_sigm(b[0][i] + vr[i]), ug = gru_sigm(b[1][i] + vu[i]);
            o[i] = ug * b[3][i] + (1.f - ug) * gru_tanh(rg * vx[i] + b[2][i]);
          }
          if (valid) {
            st8(s1 + 8 * c, o);
            gru_store4(xo + 8 * c, ep.lo_x, o[0], o[1], o[2], o[3]);
            gru_store4(xo + 8 * c + 4, ep.lo_x, o[4], o[5], o[6], o[7]);
          }
        }
      } else if constexpr (EPI == EPI_GRU2) {
        // this warp's group: units j0..j0+31; D1 = [hx | r | u] (s1 range), D2 = [r | u | cx] (c range)
        const int j0 = (colbase >> 7) * 32;
        const uint32_t t1 = tmem + ((uint32_t)(q * 32) << 16) + 96 * half, t2 = t1 + 192;
        float* so = nullptr;
        if (valid) {
          const int dst = ep.row_dst[grow];
          if (dst >= 0) so = (ep.gs ? ep.gs[ep.row_grp[grow]].S : ep.Sout) + (int64_t)dst * ep.Hp + j0;
        }
        __nv_bfloat16* xo = ep.X + (int64_t)grow * ep.ldx + ep.x_col + j0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float hx[8], r1[8], u1[8], r2[8], u2[8], cx8[8];
          tmem_ld8_nowait(t1 + 8 * c, hx);
          tmem_ld8_nowait(t1 + 32 + 8 * c, r1);
          tmem_ld8_nowait(t1 + 64 + 8 * c, u1);
          tmem_ld8_nowait(t2 + 8 * c, r2);
          tmem_ld8_nowait(t2 + 32 + 8 * c, u2);
          tmem_ld8_nowait(t2 + 64 + 8 * c, cx8);
          tmem_wait_ld();
          reg_dep8(hx); reg_dep8(r1); reg_dep8(u1); reg_dep8(r2); reg_dep8(u2); reg_dep8(cx8);
          float(&bb)[3][8] = bia[c & 1];
          if (valid) {
            float o[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float rg = gru_sigm((r1[i] + r2[i]) + bb[0][i]), ug = gru_sigm((u1[i] + u2[i]) + bb[1][i]);
              o[i] = ug * s1in[c][i] + (1.f - ug) * gru_tanh(rg * (hx[i] + bb[2][i]) + cx8[i]);
            }
            if (so) st8(so + 8 * c, o);
            gru_store4(xo + 8 * c, ep.lo_x, o[0], o[1], o[2], o[3]);
            gru_store4(xo + 8 * c + 4, ep.lo_x, o[4], o[5], o[6], o[7]);
          }
          if (c + 2 < 4) bias_fetch(c + 2, bia[c & 1]);
        }
      } else if constexpr (EPI == EPI_READOUT) {
        static_assert(COLS == 64 || COLS == 32, "EPI_READOUT: 64 or 32 readout columns per epilogue warp");
        // (tcgen05.ld / wait are warp-collective: every lane loads, only valid rows write)
        int dst = -1;
        if (valid) dst = ep.row_dst[grow];
        float* tr = dst >= 0 ? (ep.gs ? ep.gs[ep.row_grp[grow]].T : ep.Tout) + (int64_t)dst * ep.Ep : nullptr;
        __nv_bfloat16* at = ep.A_t + (int64_t)grow * ep.lda_t;
        const int E = ep.E;
        // 8 outputs t[k0 .. k0 + 8) per pass: maxout pairs columns (2k, 2k + 1) (16 columns), tanh 8
        auto emit = [&](int k0, float(&t)[8]) {
          float hi[8], lo[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int k = k0 + i;
            t[i] = k < E ? t[i] : 0.f;  // (t -> arena, zero past E)
            const float av = k < E ? t[i] : ((k == E || (k == E + 1 && ep.lo_t == 0)) ? 1.f : 0.f);
            hi[i] = av;
            lo[i] = k < E ? av - __bfloat162float(__float2bfloat16_rn(av)) : 0.f;  // (bias columns: lo 0)
          }
          if (tr && k0 < ep.Ep) st8(tr + k0, t);
          if (k0 < ep.Ep) {
            *reinterpret_cast<uint4*>(at + k0) = make_uint4(gru_pk(hi[0], hi[1]), gru_pk(hi[2], hi[3]),
                                                            gru_pk(hi[4], hi[5]), gru_pk(hi[6], hi[7]));
            if (ep.lo_t > 0)
              *reinterpret_cast<uint4*>(at + ep.lo_t + k0) = make_uint4(gru_pk(lo[0], lo[1]), gru_pk(lo[2], lo[3]),
                                                                        gru_pk(lo[4], lo[5]), gru_pk(lo[6], lo[7]));
          }
        };
        if (ep.maxout) {
#pragma unroll
          for (int ps = 0; ps < COLS / 16; ++ps) {
            float a[16], t[8];
            tmem_ld8_nowait(tbase + 16 * ps, a);
            tmem_ld8_nowait(tbase + 16 * ps + 8, a + 8);
            tmem_wait_ld();
            reg_dep8(a);
            reg_dep8(a + 8);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float* e = epj[(16 * ps + 2 * i) / 8];
              const int o = (2 * i) % 8;
              t[i] = fmaxf(a[2 * i] + e[o], a[2 * i + 1] + e[o + 1]);
            }
            if (valid) emit(colbase / 2 + 8 * ps, t);
          }
        } else {
#pragma unroll
          for (int ps = 0; ps < COLS / 8; ++ps) {
            float a[8], t[8];
            tmem_ld8_nowait(tbase + 8 * ps, a);
            tmem_wait_ld();
            reg_dep8(a);
#pragma unroll
            for (int i = 0; i < 8; ++i) t[i] = gru_tanh(a[i] + epj[ps][i]);
            if (valid) emit(colbase + 8 * ps, t);
          }
        }
      } else {  // EPI_LSE: online (max, sum exp, argmax) over this warp's COLS logits of the row
#pragma unroll 1
        for (int c = 0; c < COLS; c += 64) {
          float v[64];
          tmem_ld32_nowait(tbase + c, v);
          tmem_ld32_nowait(tbase + c + 32, v + 32);
          tmem_wait_ld_dep(v);
          reg_dep32(v + 32);
          const int col0 = colbase + c + g.n_off;
          if (col0 + 64 > ep.n_valid) {  // padded vocabulary columns (last tile only)
#pragma unroll
            for (int j = 0; j < 64; ++j)
              if (col0 + j >= ep.n_valid) v[j] = -INFINITY;
          }
          float t32[32];  // tree max
#pragma unroll
          for (int j = 0; j < 32; ++j) t32[j] = fmaxf(v[j], v[j + 32]);
#pragma unroll
          for (int k = 16; k > 0; k >>= 1)
#pragma unroll
            for (int j = 0; j < k; ++j) t32[j] = fmaxf(t32[j], t32[j + k]);
          const float cm = t32[0];
          if (cm > mx) {  // new running max (rare after the first chunks): lowest index of it
            int ix[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) ix[j] = v[j] == cm ? j : (v[j + 32] == cm ? j + 32 : 64);
#pragma unroll
            for (int k = 16; k > 0; k >>= 1)
#pragma unroll
              for (int j = 0; j < k; ++j) ix[j] = min(ix[j], ix[j + k]);
            const float f = ex2_approx((mx - cm) * LOG2E);
            s0 *= f; s1 *= f; s2 *= f; s3 *= f;
            mx = cm;
            am = col0 + ix[0];
          }
          if (mx > -INFINITY) {
            const float mb = mx * LOG2E;
#pragma unroll
            for (int j = 0; j < 64; j += 4) {
              s0 += ex2_approx(fmaf(v[j], LOG2E, -mb));
              s1 += ex2_approx(fmaf(v[j + 1], LOG2E, -mb));
              s2 += ex2_approx(fmaf(v[j + 2], LOG2E, -mb));
              s3 += ex2_approx(fmaf(v[j + 3], LOG2E, -mb));
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&tempty[acc]);
        else mbar_arrive_cluster(tempty0 + acc * 8);
      }
    }
    if constexpr (EPI == EPI_LSE) {  // one partial per (row, run, half); empty runs give (-inf, 0)
      if (valid)
        ep.part[((size_t)grow * sc.cpm + itm.c) * 2 + half] =
            make_float4(mx, (s0 + s1) + (s2 + s3), __int_as_float(am), 0.f);
    }
    if constexpr (EPI == EPI_TOPK) {  // kTopK (logit, column) per (row, run, half)
      if (valid) {
        float2* dst = ep.topk + (((size_t)grow * sc.cpm + itm.c) * 2 + half) * kTopK;
#pragma unroll
        for (int q = 0; q < kTopK; ++q) dst[q] = make_float2(tv[q], __int_as_float(ti[q]));
      }
    }
  }
}

template <int BN, int STAGES, int EPI, bool PAIR, bool ARES = false>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
           const __grid_constant__ CUtensorMap tmC, GemmShape g, EpiParams ep) {
  extern __shared__ uint8_t smem_raw[];
  GemmCta<BN, STAGES, EPI, PAIR, ARES> cx;
  cx.carve(smem_raw);
  if (threadIdx.x == 0) GTRACE(0);
  if (cx.warp == 0 && cx.lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (EPI == EPI_STORE || g.b2_kb1 > 0) tma_prefetch(&tmC);
  }
  cx.setup();
  if (threadIdx.x == 0) GTRACE(1);
  pdl_enter();  // prologue above overlaps the previous kernel; inputs (and M_dev) are read below
  if (threadIdx.x == 0) GTRACE(2);
  constexpr int CM = GemmCta<BN, STAGES, EPI, PAIR, ARES>::CM;
  const int M = g.M_dev ? *g.M_dev : g.M;
  const Sched sc = make_sched<EPI>(g, M, CM, BN, cx.nunits);
  if ((EPI == EPI_LSE || EPI == EPI_TOPK) && blockIdx.x == 0 && threadIdx.x == 0 && ep.cpm_out) *ep.cpm_out = sc.cpm;
  if (cx.warp == 0) {
    gemm_produce(cx, &tmA, &tmB, &tmC, g, sc);  // (whole warp; tmC = the second B operand when b2_kb1 > 0)
  } else if (cx.warp == 1) {
    if (cx.leader) gemm_mma(cx, g, sc, ep);  // (whole warp)
  } else {
    gemm_epilogue(cx, &tmC, g, M, sc, ep);
  }
  if (EPI == EPI_STORE && cx.warp >= 2 && cx.lane == 0) bulk_wait_all();
  if (cx.warp == 2 && cx.lane == 0) GTRACE(6);
  cx.teardown();
  if (threadIdx.x == 0) GTRACE(7);
}

// ------------------------------------------------------------------------------------- host side
typedef CUresult (*PFN_tmapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                         const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                         CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                         CUtensorMapFloatOOBfill);

static PFN_tmapEncodeTiled get_encode_fn() {
  static PFN_tmapEncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_tmapEncodeTiled>(p);
  });
  if (!fn) throw NmtError(NMT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap make_tmap_bf16(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw NmtError(NMT_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ") rows=" +
                                     std::to_string(rows) + " cols=" + std::to_string(cols));
  return m;
}

// fp32 output map for the TMA-store epilogue: box 32 x 32, 128B swizzle; cached per buffer
static CUtensorMap make_tmap_f32_out(const void* base, uint64_t rows, uint64_t cols) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw NmtError(NMT_ERR_CUDA, "cuTensorMapEncodeTiled (fp32 out) failed");
  return m;
}
static const CUtensorMap& out_map(const float* out, uint64_t rows, uint64_t ldc) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, uint64_t, uint64_t>, CUtensorMap> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple((const void*)out, rows, ldc);
  auto it = cache.find(key);
  if (it == cache.end()) it = cache.emplace(key, make_tmap_f32_out(out, rows, ldc)).first;
  return it->second;
}

template <int BN, int STAGES, int EPI, bool PAIR, bool ARES = false>
static void launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const GemmShape& g,
                   const EpiParams& ep, int M_max, cudaStream_t st) {
  using S = GemmSmem<BN, STAGES, EPI, PAIR, ARES>;
  static_assert(S::BYTES <= 232448, "shared memory budget");
  static std::atomic<size_t> smem_attr[kMaxDevices];  // per template instance and device
  ensure_smem_attr(k_gemm<BN, STAGES, EPI, PAIR, ARES>, smem_attr, (size_t)S::BYTES);
  const int CM = PAIR ? 2 * BM : BM;
  int tiles = 0;  // work items at M_max rows (EPI_STORE: per region, with its split count)
  for (int r = 0, nt0 = 0; r < g.nreg; ++r) {
    const int nt1 = r < g.nreg - 1 ? g.reg_n_end[r] / BN : g.N / BN;
    tiles += ((M_max + CM - 1) / CM) * (nt1 - nt0) * gemm_ks(g, r);
    nt0 = nt1;
  }
  int grid = (PAIR ? 2 : 1) * tiles;
  if (EPI == EPI_LSE || EPI == EPI_TOPK || grid > kNumSMs) grid = kNumSMs;  // persistent (LSE / TOPK runs use every unit)
  if (grid <= 0) return;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = S::BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = PAIR ? 2 : 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = PAIR ? 2 : 1;
#ifdef NMT_DIAG
  if (getenv("NMT_GEMM_TRACE")) {  // (diagnostic) serialise, stamp every CTA's phases, print a summary
    EpiParams et = ep;
    CK(cudaMalloc(&et.trace, (size_t)grid * 8 * 8));
    CK(cudaMemsetAsync(et.trace, 0, (size_t)grid * 8 * 8, st));
    CK(cudaLaunchKernelEx(&cfg, k_gemm<BN, STAGES, EPI, PAIR, ARES>, a, b, c, g, et));
    CK_LAUNCH();
    std::vector<unsigned long long> h((size_t)grid * 8);
    CK(cudaMemcpyAsync(h.data(), et.trace, h.size() * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    cudaFree(et.trace);
    unsigned long long t0 = ~0ull;
    for (int i = 0; i < grid; ++i) t0 = std::min(t0, h[(size_t)i * 8]);
    fprintf(stderr, "[gemm_trace] BN=%d ST=%d EPI=%d PAIR=%d grid=%d nreg=%d ks=%d us from first entry (min/med/max):", BN,
            STAGES, EPI, (int)PAIR, grid, g.nreg, g.ksplit);
    for (int ev = 0; ev < 8; ++ev) {
      std::vector<double> v;
      for (int i = 0; i < grid; ++i)
        if (h[(size_t)i * 8 + ev]) v.push_back((double)(h[(size_t)i * 8 + ev] - t0) * 1e-3);
      if (v.empty()) continue;
      std::sort(v.begin(), v.end());
      fprintf(stderr, " e%d %.1f/%.1f/%.1f", ev, v.front(), v[v.size() / 2], v.back());
    }
    fprintf(stderr, "\n");
    return;
  }
#endif
  CK(cudaLaunchKernelEx(&cfg, k_gemm<BN, STAGES, EPI, PAIR, ARES>, a, b, c, g, ep));
  CK_LAUNCH();
}

void gemm_validate(const GemmShape& g, int BN) {
  if (g.N % BN) throw NmtError(NMT_ERR_INVALID_ARG, "gemm: N not a multiple of the N tile");
  if (g.ksplit < 1) throw NmtError(NMT_ERR_INVALID_ARG, "gemm: ksplit < 1");
  for (int r = 0; r < g.nreg; ++r) {  // every split must own >= 1 k-block of its region
    const int ks = gemm_ks(g, r);
    if (ks < 1) throw NmtError(NMT_ERR_INVALID_ARG, "gemm: region split < 1");
    const int nkb = g.passes * (g.reg_k1[r] - g.reg_k0[r]) / BK;
    const int chunk = (nkb + ks - 1) / ks;
    if ((ks - 1) * chunk >= nkb) throw NmtError(NMT_ERR_INVALID_ARG, "gemm: empty K split");
  }
  for (int r = 0; r < g.nreg; ++r) {
    if (g.reg_k0[r] % BK || g.reg_k1[r] % BK || g.reg_k1[r] <= g.reg_k0[r])
      throw NmtError(NMT_ERR_INVALID_ARG, "gemm: bad K region");
    if (r < g.nreg - 1 && g.reg_n_end[r] % BN) throw NmtError(NMT_ERR_INVALID_ARG, "gemm: region not tile aligned");
  }
}

// fp32 output GEMM (TMA-store epilogue); BN = 128 (more CTAs for the mid-size decoder GEMMs).
// out_rows = rows of the output allocation (stores are clipped there); split-K partial s goes to
// rows s * split_stride / ldc + r of the same 2-D map.
static EpiParams store_params(const GemmShape& g, int BN, float* out, int ldc, const float* bias,
                              size_t split_stride) {
  gemm_validate(g, BN);
  if (gemm_ks_max(g) > 1 && (bias || !split_stride))
    throw NmtError(NMT_ERR_INVALID_ARG, "gemm: split-K partials take no bias");
  if (split_stride % ldc) throw NmtError(NMT_ERR_INVALID_ARG, "gemm: split stride not a whole number of rows");
  EpiParams ep{};
  ep.out = out;
  ep.ldc = ldc;
  ep.bias = bias;
  ep.split_stride = split_stride;
  ep.rows_per_split = (int)(split_stride / ldc);
  return ep;
}
void gemm_store(const CUtensorMap& a, const CUtensorMap& b, const GemmShape& g, float* out, int ldc, int out_rows,
                const float* bias, int M_max, cudaStream_t st, size_t split_stride) {
  const EpiParams ep = store_params(g, 128, out, ldc, bias, split_stride);
  launch<128, 4, EPI_STORE, false>(a, b, out_map(out, out_rows, ldc), g, ep, M_max, st);
}

// fp32 output GEMM with 128 x 256 tiles (A reuse x2; fewer tiles)
void gemm_store256(const CUtensorMap& a, const CUtensorMap& b, const GemmShape& g, float* out, int ldc, int out_rows,
                   const float* bias, int M_max, cudaStream_t st, size_t split_stride) {
  const EpiParams ep = store_params(g, 256, out, ldc, bias, split_stride);
  launch<256, 3, EPI_STORE, false>(a, b, out_map(out, out_rows, ldc), g, ep, M_max, st);
}

// fp32 output GEMM on CTA pairs: 256 x 256 tiles; `b_half` = tensor map of B with a 128-row box
void gemm_store_pair(const CUtensorMap& a, const CUtensorMap& b_half, const GemmShape& g, float* out, int ldc,
                     int out_rows, const float* bias, int M_max, cudaStream_t st, size_t split_stride) {
  const EpiParams ep = store_params(g, 256, out, ldc, bias, split_stride);
  launch<256, 5, EPI_STORE, true>(a, b_half, out_map(out, out_rows, ldc), g, ep, M_max, st);
}

// fp32 output GEMM on CTA pairs with 256 x 128 tiles (measurement / engine check of the BN = 128 pair shape)
void gemm_store_pair128(const CUtensorMap& a, const CUtensorMap& b_q, const GemmShape& g, float* out, int ldc,
                        int out_rows, const float* bias, int M_max, cudaStream_t st, size_t split_stride) {
  const EpiParams ep = store_params(g, 128, out, ldc, bias, split_stride);
  launch<128, 6, EPI_STORE, true>(a, b_q, out_map(out, out_rows, ldc), g, ep, M_max, st);
}

// fused vocabulary GEMM + online log-sum-exp partials; BN = 256.
void gemm_gru_pair(const CUtensorMap& a, const CUtensorMap& b_half, const GemmShape& g, const EpiParams& ep, int M_max,
                   cudaStream_t st) {
  gemm_validate(g, 256);
  if (gemm_ks_max(g) != 1) throw NmtError(NMT_ERR_INVALID_ARG, "gemm: the fused GRU epilogue needs the full K sum");
  launch<256, 5, EPI_GRU, true>(a, b_half, b_half /*unused*/, g, ep, M_max, st);
}

static void check_b2(const GemmShape& g, const CUtensorMap* b2) {
  if (g.b2_kb1 > 0 && (!b2 || g.b2_kb0 >= g.b2_kb1 || g.b_panel_rows))
    throw NmtError(NMT_ERR_INVALID_ARG, "gemm: bad second B operand range");
}

// `b2` (or null): second B operand for k-blocks [g.b2_kb0, g.b2_kb1) (projected-context step)
void gemm_gru2_pair(const CUtensorMap& a, const CUtensorMap& b_half, const GemmShape& g, const EpiParams& ep, int M_max,
                    cudaStream_t st, const CUtensorMap* b2) {
  gemm_validate(g, 256);
  if (gemm_ks_max(g) != 1 || g.nreg != 1 || ep.Hp % BK)
    throw NmtError(NMT_ERR_INVALID_ARG, "gemm: the fused GRU2 epilogue needs the full K sum in one region");
  check_b2(g, b2);
  launch<256, 5, EPI_GRU2, true>(a, b_half, b2 ? *b2 : b_half, g, ep, M_max, st);
}

void gemm_readout_pair(const CUtensorMap& a, const CUtensorMap& b_q, const GemmShape& g, const EpiParams& ep, int M_max,
                       cudaStream_t st, const CUtensorMap* b2) {
  gemm_validate(g, 128);
  if (gemm_ks_max(g) != 1 || g.nreg != 1)
    throw NmtError(NMT_ERR_INVALID_ARG, "gemm: the fused readout epilogue needs the full K sum in one region");
  check_b2(g, b2);
  launch<128, 8, EPI_READOUT, true>(a, b_q, b2 ? *b2 : b_q, g, ep, M_max, st);
}

// the same on 256 x 64 CTA-pair tiles (`b_e` / `b2`: maps with 32-row boxes): twice the CTAs of the 256 x 128
// shape for the readout's narrow N (ROp = 1024 at E = 500: 4 x 16 pair tiles = 128 CTAs at R = 1024)
void gemm_readout_pair64(const CUtensorMap& a, const CUtensorMap& b_e, const GemmShape& g, const EpiParams& ep,
                         int M_max, cudaStream_t st, const CUtensorMap* b2) {
  gemm_validate(g, 64);
  if (gemm_ks_max(g) != 1 || g.nreg != 1)
    throw NmtError(NMT_ERR_INVALID_ARG, "gemm: the fused readout epilogue needs the full K sum in one region");
  check_b2(g, b2);
  launch<64, 10, EPI_READOUT, true>(a, b_e, b2 ? *b2 : b_e, g, ep, M_max, st);
}

void gemm_lse(const CUtensorMap& a, const CUtensorMap& b, const GemmShape& g, float4* part, int n_valid, int M_max,
              cudaStream_t st, int* cpm_out) {
  gemm_validate(g, 256);
  EpiParams ep{};
  ep.part = part;
  ep.n_valid = n_valid;
  ep.n_tiles = g.N / 256;
  ep.cpm_out = cpm_out;
  launch<256, 4, EPI_LSE, false>(a, b, b /*unused*/, g, ep, M_max, st);
}

// vocabulary GEMM + LSE on CTA pairs; `b_half` = tensor map of B with a 128-row box
// vocabulary GEMM with the top-kTopK epilogue (beam step) on CTA pairs; partials [R][2 cpm][kTopK]
void gemm_topk_pair(const CUtensorMap& a, const CUtensorMap& b_half, const GemmShape& g, float2* topk, int n_valid,
                    cudaStream_t st, int* cpm_out) {
  gemm_validate(g, 256);
  EpiParams ep{};
  ep.topk = topk;
  ep.n_valid = n_valid;
  ep.n_tiles = g.N / 256;
  ep.cpm_out = cpm_out;
  const bool ares = g.passes == 1 && g.nreg == 1 && g.ksplit == 1 && (g.reg_k1[0] - g.reg_k0[0]) <= kAresKB * BK;
  if (ares) launch<256, 6, EPI_TOPK, true, true>(a, b_half, b_half /*unused*/, g, ep, kNumSMs * BM, st);  // (as LSE)
  else launch<256, 6, EPI_TOPK, true>(a, b_half, b_half /*unused*/, g, ep, kNumSMs * BM, st);
}

void gemm_lse_pair(const CUtensorMap& a, const CUtensorMap& b_half, const GemmShape& g, float4* part, int n_valid,
                   cudaStream_t st, int* cpm_out) {
  gemm_validate(g, 256);
  EpiParams ep{};
  ep.part = part;
  ep.n_valid = n_valid;
  ep.n_tiles = g.N / 256;
  ep.cpm_out = cpm_out;
  // single-pass bf16 with K <= 512: the A tile stays resident for the unit's whole n-run (one L2 read of A
  // per item instead of one per n-tile: half the L2 -> SM bytes of the kernel)
  const bool ares = g.passes == 1 && g.nreg == 1 && g.ksplit == 1 && (g.reg_k1[0] - g.reg_k0[0]) <= kAresKB * BK;
#ifdef NMT_DIAG
  if (getenv("NMT_VOCAB_NOARES")) {
    launch<256, 6, EPI_LSE, true>(a, b_half, b_half /*unused*/, g, ep, kNumSMs * BM, st);
    return;
  }
#endif
  if (ares) launch<256, 6, EPI_LSE, true, true>(a, b_half, b_half /*unused*/, g, ep, kNumSMs * BM, st);
  else launch<256, 6, EPI_LSE, true>(a, b_half, b_half /*unused*/, g, ep, kNumSMs * BM, st);
}

}  // namespace nmt
