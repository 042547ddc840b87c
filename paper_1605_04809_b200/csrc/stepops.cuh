// stepops.cuh - elementwise pieces of the decoder step shared by their standalone kernels (kernels.cu)
// and the chained decoder-tail GEMM kernel (gemm.cu): GRU2 gates (D6) and the readout (D7).
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace nmt {

// Elementwise step kernels: one thread per (row, 4 consecutive hidden units), float4 loads all
// issued before any math (latency-bound otherwise); rows r >= *R exit.
NMT_DEV float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
NMT_DEV void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
NMT_DEV uint32_t pk_bf16(float a, float b) {
  uint32_t y;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(b), "f"(a));
  return y;
}
// write 4 values as bf16 hi (and the bf16 lo residuals at +lo_off) - 8-byte stores
NMT_DEV void store_split4(__nv_bfloat16* hi, int lo_off, float4 v) {
  const uint32_t h01 = pk_bf16(v.x, v.y), h23 = pk_bf16(v.z, v.w);
  *reinterpret_cast<uint2*>(hi) = make_uint2(h01, h23);
  if (lo_off > 0) {
    const float r0 = v.x - __uint_as_float(h01 << 16), r1 = v.y - __uint_as_float(h01 & 0xffff0000u);
    const float r2 = v.z - __uint_as_float(h23 << 16), r3 = v.w - __uint_as_float(h23 & 0xffff0000u);
    *reinterpret_cast<uint2*>(hi + lo_off) = make_uint2(pk_bf16(r0, r1), pk_bf16(r2, r3));
  }
}
NMT_DEV float sigm(float x) { return 1.f / (1.f + expf(-x)); }

// sum of the split-K partials of a decoder GEMM output, in split order (deterministic)
NMT_DEV float4 ld4_sum(const float* p, int ks, int64_t stride) {
  float4 a = ld4(p);
  for (int s = 1; s < ks; ++s) {
    const float4 b = ld4(p + s * stride);
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
  }
  return a;
}
NMT_DEV float ld_sum(const float* p, int ks, int64_t stride) {
  float a = p[0];
  for (int s = 1; s < ks; ++s) a += p[s * stride];
  return a;
}


// D6: GRU2 gates.  G2 = [s1 U_nl + c Wc | s1 Ux_nl | c Wcx] (one region GEMM).
NMT_DEV void gru2_elem(const StepDev& d, float* __restrict__ S, int idx) {
  const int Hp = d.Hp, H4 = (d.H + 3) / 4;
  const int r = idx / H4, j = (idx % H4) * 4;
  if (r >= *d.R) return;
  const float* g = d.G2 + (int64_t)r * 4 * Hp + j;
  const float4 gr = ld4_sum(g, d.ks_g2[0], d.ps_g2), gu = ld4_sum(g + Hp, d.ks_g2[0], d.ps_g2),
               gh = ld4_sum(g + 2 * Hp, d.ks_g2[1], d.ps_g2), gc = ld4_sum(g + 3 * Hp, d.ks_g2[2], d.ps_g2);
  const float4 br = ld4(d.b_nl + j), bu = ld4(d.b_nl + Hp + j), bx = ld4(d.bx_nl + j);
  const float4 s1 = ld4(d.S1 + (int64_t)r * Hp + j);
  float4 o;
#define NMT_GRU2(c) { const float rg = sigm(gr.c + br.c), ug = sigm(gu.c + bu.c); \
                      o.c = ug * s1.c + (1.f - ug) * tanhf(rg * (gh.c + bx.c) + gc.c); }
  NMT_GRU2(x) NMT_GRU2(y) NMT_GRU2(z) NMT_GRU2(w)
#undef NMT_GRU2
  const int dst = d.row_dst[r];
  if (dst >= 0) st4((d.gs ? d.gs[d.row_grp[r]].S : S) + (int64_t)dst * Hp + j, o);
  store_split4(d.X + (int64_t)r * d.ldx + d.Hp + d.Cp + j, d.lo_x, o);
}

// Row r, columns k..k+3 of the bf16 A operand of the vocabulary GEMM from t (zero past E): the two
// bias columns (b_o folded into the GEMM as hi + lo) are 1 at E (and E+1 in single pass); in split
// mode the lo half carries t - bf16(t) and 0 in the bias columns.
NMT_DEV void write_vocab_operand(const StepDev& d, int r, int k, const float (&tp)[4]) {
  const int E = d.E;
  float4 av;
  float* ap = &av.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int kk = k + i;
    ap[i] = kk < E ? tp[i] : ((kk == E || (kk == E + 1 && d.lo_t == 0)) ? 1.f : 0.f);
  }
  __nv_bfloat16* at = d.A_t + (int64_t)r * d.lda_t + k;
  if (k + 3 < E || d.lo_t == 0) {
    store_split4(at, d.lo_t, av);
  } else {  // split path, bias columns: hi = 1 at E, lo part of the bias columns = 0
    store_split4(at, 0, av);
    const float4 lo4 = make_float4(k < E ? tp[0] - __bfloat162float(__float2bfloat16_rn(tp[0])) : 0.f,
                                   k + 1 < E ? tp[1] - __bfloat162float(__float2bfloat16_rn(tp[1])) : 0.f,
                                   k + 2 < E ? tp[2] - __bfloat162float(__float2bfloat16_rn(tp[2])) : 0.f,
                                   k + 3 < E ? tp[3] - __bfloat162float(__float2bfloat16_rn(tp[3])) : 0.f);
    const uint32_t l01 = pk_bf16(lo4.x, lo4.y), l23 = pk_bf16(lo4.z, lo4.w);
    *reinterpret_cast<uint2*>(at + d.lo_t) = make_uint2(l01, l23);
  }
}

// D7: readout activation.  RO = c W_ctx + s2 W_l (GEMM), Ep[y] = e W_p + b_p + b_l + b_ctx.
// Writes t (fp32) to the arena and the bf16 A operand of the vocabulary GEMM with the two
// bias columns (b_o folded into the GEMM as hi + lo).  Thread per (row, 4 outputs).
NMT_DEV void readout_elem(const StepDev& d, float* __restrict__ T, int idx) {
  const int E = d.E, Ep = d.Ep, E4 = Ep / 4;
  const int r = idx / E4, k = (idx % E4) * 4;
  if (r >= *d.R) return;
  const int dst = d.row_dst[r];
  const int y = dst >= 0 ? d.row_y[r] : -1;
  const float* pre = d.RO + (int64_t)r * d.ROp;
  const float* epr = d.Eproj + (int64_t)(y < 0 ? d.V : y) * d.ROp;
  float t[4];
  if (d.maxout) {
    if (2 * k + 7 < d.ROp) {
      const float4 a0 = ld4_sum(pre + 2 * k, d.ks_ro, d.ps_ro), a1 = ld4_sum(pre + 2 * k + 4, d.ks_ro, d.ps_ro);
      const float4 b0 = ld4(epr + 2 * k), b1 = ld4(epr + 2 * k + 4);
      t[0] = fmaxf(a0.x + b0.x, a0.y + b0.y);
      t[1] = fmaxf(a0.z + b0.z, a0.w + b0.w);
      t[2] = fmaxf(a1.x + b1.x, a1.y + b1.y);
      t[3] = fmaxf(a1.z + b1.z, a1.w + b1.w);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        t[i] = k + i < E ? fmaxf(ld_sum(pre + 2 * (k + i), d.ks_ro, d.ps_ro) + epr[2 * (k + i)],
                                 ld_sum(pre + 2 * (k + i) + 1, d.ks_ro, d.ps_ro) + epr[2 * (k + i) + 1]) : 0.f;
    }
  } else {
    if (k + 3 < d.ROp) {
      const float4 a = ld4_sum(pre + k, d.ks_ro, d.ps_ro), b = ld4(epr + k);
      t[0] = tanhf(a.x + b.x); t[1] = tanhf(a.y + b.y); t[2] = tanhf(a.z + b.z); t[3] = tanhf(a.w + b.w);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) t[i] = k + i < E ? tanhf(ld_sum(pre + k + i, d.ks_ro, d.ps_ro) + epr[k + i]) : 0.f;
    }
  }
  float tp[4];  // t -> arena (zero past E)
#pragma unroll
  for (int i = 0; i < 4; ++i) tp[i] = k + i < E ? t[i] : 0.f;
  if (dst >= 0) st4((d.gs ? d.gs[d.row_grp[r]].T : T) + (int64_t)dst * Ep + k, make_float4(tp[0], tp[1], tp[2], tp[3]));
  write_vocab_operand(d, r, k, tp);
}



}  // namespace nmt
