// randparams.cpp - seeded synthetic model generator behind nmt_random_params / nmt_create_random
// (SURVEY §8(d) "Synthetic model generator").  Host C++, no model arithmetic: it only
// draws numbers and writes the params container (include/nmt.h "Params container").
//
// Distributions (the same recipe as synth/ in numpy; NOT the same numbers - the two generators are
// never assumed to agree bit for bit, a model made here is compared through its saved container):
//   embeddings ~ N(0, 1); linear maps ~ N(0, 1/fan_in); biases (incl. c_tt) ~ N(0, 0.1^2);
//   recurrent U, Ux, U_nl, Ux_nl: orthogonal H x H blocks (DL4MT ortho_weight: Q of the QR of a
//   Gaussian matrix with diag(R) > 0, i.e. Haar-distributed); U_att ~ N(0, (2/sqrt(2H))^2);
//   W_o ~ N(0, sigma^2), sigma = logit_std / sqrt(E * m2) with m2 = 0.6 (tanh) / 3.0 (maxout);
//   b_o[w] = -ln(w + 1) (Zipf prior).
// Random numbers: counter-based.  Array a (its name hashed with FNV-1a) and element i give
//   u = (splitmix64(key_a ^ splitmix64(2i + j)) >> 11 + 0.5) * 2^-53,  j in {0, 1},
// and a normal deviate by Box-Muller, so every element is independent of the draw order and the
// arrays can be generated in parallel.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/nmt.h"

namespace {

uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001b3ULL;
  }
  return h;
}

struct Stream {
  uint64_t key;
  double uniform(uint64_t ctr) const {
    return ((double)(splitmix64(key ^ splitmix64(ctr)) >> 11) + 0.5) * (1.0 / 9007199254740992.0);
  }
  double normal(uint64_t i) const {  // Box-Muller, cosine branch
    const double u1 = uniform(2 * i), u2 = uniform(2 * i + 1);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925 * u2);
  }
};

struct Spec {
  std::string name;
  int rows, cols;
};

std::vector<Spec> shapes(const nmt_dims& d) {
  const int E = d.dim_emb, H = d.dim_hid, C = 2 * H, RO = d.readout == NMT_READOUT_MAXOUT ? 2 * E : E;
  std::vector<Spec> s = {{"Wemb", d.vocab_src, E}, {"Wemb_dec", d.vocab_tgt, E}};
  for (std::string p : {"encoder", "encoder_r"}) {
    s.push_back({p + "_W", E, 2 * H});
    s.push_back({p + "_b", 1, 2 * H});
    s.push_back({p + "_U", H, 2 * H});
    s.push_back({p + "_Wx", E, H});
    s.push_back({p + "_bx", 1, H});
    s.push_back({p + "_Ux", H, H});
  }
  const std::vector<Spec> rest = {
      {"ff_state_W", C, H},        {"ff_state_b", 1, H},          {"decoder_W", E, 2 * H},
      {"decoder_b", 1, 2 * H},     {"decoder_U", H, 2 * H},       {"decoder_Wx", E, H},
      {"decoder_bx", 1, H},        {"decoder_Ux", H, H},          {"decoder_U_nl", H, 2 * H},
      {"decoder_b_nl", 1, 2 * H},  {"decoder_Ux_nl", H, H},       {"decoder_bx_nl", 1, H},
      {"decoder_Wc", C, 2 * H},    {"decoder_Wcx", C, H},         {"decoder_W_comb_att", H, C},
      {"decoder_Wc_att", C, C},    {"decoder_b_att", 1, C},       {"decoder_U_att", C, 1},
      {"decoder_c_tt", 1, 1},      {"ff_logit_lstm_W", H, RO},    {"ff_logit_lstm_b", 1, RO},
      {"ff_logit_prev_W", E, RO},  {"ff_logit_prev_b", 1, RO},    {"ff_logit_ctx_W", C, RO},
      {"ff_logit_ctx_b", 1, RO},   {"ff_logit_W", E, d.vocab_tgt}, {"ff_logit_b", 1, d.vocab_tgt}};
  s.insert(s.end(), rest.begin(), rest.end());
  return s;
}

bool ends_with(const std::string& s, const char* t) {
  const size_t n = std::strlen(t);
  return s.size() >= n && s.compare(s.size() - n, n, t) == 0;
}

// columns [col0, col0 + n) of the row-major [n x ld] array `out` := Q of a Gaussian n x n matrix
// (modified Gram-Schmidt, re-orthogonalised once; diag(R) > 0 by construction)
void ortho_block(const Stream& g, uint64_t ctr0, int n, float* out, int ld, int col0) {
  std::vector<double> q((size_t)n * n);  // column j stored contiguously at q[j * n]
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) q[(size_t)j * n + k] = g.normal(ctr0 + (uint64_t)k * n + j);
  for (int j = 0; j < n; ++j) {
    double* v = &q[(size_t)j * n];
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i < j; ++i) {
        const double* u = &q[(size_t)i * n];
        double dot = 0;
        for (int k = 0; k < n; ++k) dot += u[k] * v[k];
        for (int k = 0; k < n; ++k) v[k] -= dot * u[k];
      }
    double nr = 0;
    for (int k = 0; k < n; ++k) nr += v[k] * v[k];
    nr = 1.0 / std::sqrt(nr);
    for (int k = 0; k < n; ++k) v[k] *= nr;
  }
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j) out[(size_t)k * ld + col0 + j] = (float)q[(size_t)j * n + k];
}

void fill(const nmt_dims& d, uint64_t seed, float logit_std, const Spec& s, float* a) {
  const Stream g{splitmix64(seed) ^ fnv1a(s.name)};
  const int H = d.dim_hid;
  const size_t n = (size_t)s.rows * s.cols;
  if (s.name == "Wemb" || s.name == "Wemb_dec") {
    for (size_t i = 0; i < n; ++i) a[i] = (float)g.normal(i);
  } else if (ends_with(s.name, "_U") || ends_with(s.name, "_U_nl")) {
    ortho_block(g, 0, H, a, 2 * H, 0);
    ortho_block(g, (uint64_t)H * H, H, a, 2 * H, H);
  } else if (ends_with(s.name, "_Ux") || ends_with(s.name, "_Ux_nl")) {
    ortho_block(g, 0, H, a, H, 0);
  } else if (s.name == "decoder_U_att") {
    const double sd = 2.0 / std::sqrt((double)s.rows);
    for (size_t i = 0; i < n; ++i) a[i] = (float)(g.normal(i) * sd);
  } else if (s.name == "ff_logit_W") {
    const double m2 = d.readout == NMT_READOUT_MAXOUT ? 3.0 : 0.6;
    const double sd = logit_std / std::sqrt(d.dim_emb * m2);
    for (size_t i = 0; i < n; ++i) a[i] = (float)(g.normal(i) * sd);
  } else if (s.name == "ff_logit_b") {
    for (size_t i = 0; i < n; ++i) a[i] = (float)(-std::log((double)(i + 1)));
  } else if (s.rows == 1) {
    for (size_t i = 0; i < n; ++i) a[i] = (float)(g.normal(i) * 0.1);
  } else {
    const double sd = 1.0 / std::sqrt((double)s.rows);
    for (size_t i = 0; i < n; ++i) a[i] = (float)(g.normal(i) * sd);
  }
}

}  // namespace

extern "C" __attribute__((visibility("default"))) nmt_status nmt_random_params(const nmt_dims* d, uint64_t seed,
                                                                                float logit_std, void* out,
                                                                                size_t* len) {
  if (!d || !len) return NMT_ERR_INVALID_ARG;
  if (d->dim_emb <= 0 || d->dim_hid <= 0 || d->vocab_src <= 0 || d->vocab_tgt <= 0 ||
      (d->readout != NMT_READOUT_TANH && d->readout != NMT_READOUT_MAXOUT) || !(logit_std > 0.f))
    return NMT_ERR_INVALID_ARG;
  const std::vector<Spec> sp = shapes(*d);
  std::string head = "NMTPARAMS 1\ndims " + std::to_string(d->dim_emb) + " " + std::to_string(d->dim_hid) + " " +
                     std::to_string(d->vocab_src) + " " + std::to_string(d->vocab_tgt) + " readout=" +
                     (d->readout == NMT_READOUT_MAXOUT ? "maxout" : "tanh") + " eos=0 unk=1\narrays " +
                     std::to_string(sp.size()) + "\n";
  for (const Spec& s : sp) head += s.name + " " + std::to_string(s.rows) + " " + std::to_string(s.cols) + "\n";
  head.append((64 - head.size() % 64) % 64, '\0');
  size_t total = head.size();
  std::vector<size_t> at(sp.size());
  for (size_t i = 0; i < sp.size(); ++i) {
    at[i] = total;
    total += (size_t)sp[i].rows * sp[i].cols * 4;
  }
  if (!out) {
    *len = total;
    return NMT_OK;
  }
  if (*len < total) {
    *len = total;
    return NMT_ERR_CAPACITY;
  }
  char* o = static_cast<char*>(out);
  std::memcpy(o, head.data(), head.size());
  // one thread per array (the orthogonal blocks dominate: O(H^3) each)
  std::vector<std::thread> th;
  for (size_t i = 0; i < sp.size(); ++i)
    th.emplace_back([&, i] { fill(*d, seed, logit_std, sp[i], reinterpret_cast<float*>(o + at[i])); });
  for (auto& t : th) t.join();
  *len = total;
  return NMT_OK;
}
