// std::mt19937_64 with GF(2) jump-ahead (see mt64.h).
#include "mt64.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <thread>

namespace seraph::mt64 {

void seed_window(uint64_t seed, uint64_t* win) {
  win[0] = seed;
  for (int i = 1; i < kN; ++i)
    win[i] = 6364136223846793005ull * (win[i - 1] ^ (win[i - 1] >> 62)) + uint64_t(i);
}

void advance_window(uint64_t* win) {
  const uint64_t nx = twist(win[0], win[1], win[kM]);
  std::memmove(win, win + 1, (kN - 1) * sizeof(uint64_t));
  win[kN - 1] = nx;
}

void Engine::load(const uint64_t* win) {
  std::memcpy(mt, win, sizeof(mt));
  idx = kN;
}

uint64_t Engine::operator()() {
  if (idx >= kN) {
    for (int k = 0; k < kN - kM; ++k) mt[k] = twist(mt[k], mt[k + 1], mt[k + kM]);
    for (int k = kN - kM; k < kN - 1; ++k) mt[k] = twist(mt[k], mt[k + 1], mt[k + kM - kN]);
    mt[kN - 1] = twist(mt[kN - 1], mt[0], mt[kM - 1]);
    idx = 0;
  }
  return temper(mt[idx++]);
}

namespace {

// raw words x[0..len) starting from a window (x[0..311] = win)
void raw_sequence(const uint64_t* win, uint64_t* x, size_t len) {
  std::memcpy(x, win, kN * sizeof(uint64_t));
  for (size_t k = 0; k + kN < len; ++k) x[k + kN] = twist(x[k], x[k + 1], x[k + kM]);
}

inline bool bit(const std::vector<uint64_t>& v, size_t i) { return (v[i >> 6] >> (i & 63)) & 1u; }

// Berlekamp-Massey over GF(2) on 2*kDeg output bits (bit 0 of the raw words
// generated from W_0), returning the connection polynomial's reciprocal.
Poly compute_charpoly() {
  const size_t N = 2 * size_t(kDeg);
  std::vector<uint64_t> win(kN);
  seed_window(5489u, win.data());
  std::vector<uint64_t> x(N + 2 * kN);
  raw_sequence(win.data(), x.data(), x.size());
  const size_t W = (N + 127) / 64 + 2;
  // R[k] = s_{N-1-k}, s_i = bit 0 of x[kN + i]
  std::vector<uint64_t> R(W + 2, 0);
  for (size_t i = 0; i < N; ++i)
    if (x[kN + i] & 1u) R[(N - 1 - i) >> 6] |= 1ull << ((N - 1 - i) & 63);
  std::vector<uint64_t> C(W, 0), B(W, 0), T;
  C[0] = B[0] = 1;
  size_t L = 0, m = 1;
  auto xor_shifted = [&](std::vector<uint64_t>& dst, const std::vector<uint64_t>& src, size_t sh) {
    const size_t ws = sh >> 6, bs = sh & 63;
    for (size_t w = W; w-- > ws;) {
      uint64_t v = src[w - ws] << bs;
      if (bs && w - ws >= 1) v |= src[w - ws - 1] >> (64 - bs);
      dst[w] ^= v;
    }
  };
  for (size_t n = 0; n < N; ++n) {
    const size_t base = N - 1 - n, bw = base >> 6, bb = base & 63;
    uint64_t acc = 0;
    for (size_t w = 0; w <= (L >> 6); ++w) {
      uint64_t r = R[bw + w] >> bb;
      if (bb) r |= R[bw + w + 1] << (64 - bb);
      acc ^= r & C[w];
    }
    if (!(__builtin_popcountll(acc) & 1)) {
      ++m;
    } else if (2 * L <= n) {
      T = C;
      xor_shifted(C, B, m);
      L = n + 1 - L;
      B = T;
      m = 1;
    } else {
      xor_shifted(C, B, m);
      ++m;
    }
  }
  Poly phi(kPolyWords, 0);
  if (L != size_t(kDeg)) return Poly();  // never: MT19937-64 has a primitive phi
  for (size_t k = 0; k <= L; ++k)
    if (bit(C, L - k)) phi[k >> 6] |= 1ull << (k & 63);
  return phi;
}

struct Tables {
  Poly phi;
  std::vector<uint64_t> shifted;  // 64 x (kPolyWords + 1): phi << b
};

const Tables& tables() {
  static Tables t;
  static std::once_flag once;
  std::call_once(once, [] {
    t.phi = compute_charpoly();
    t.shifted.assign(64 * (kPolyWords + 1), 0);
    for (int b = 0; b < 64; ++b) {
      uint64_t* o = t.shifted.data() + size_t(b) * (kPolyWords + 1);
      for (int w = 0; w < kPolyWords; ++w) {
        o[w] |= b ? t.phi[w] << b : t.phi[w];
        if (b) o[w + 1] |= t.phi[w] >> (64 - b);
      }
    }
  });
  return t;
}

// r (2*kPolyWords words) mod phi -> first kPolyWords words
void reduce(std::vector<uint64_t>& r) {
  const Tables& t = tables();
  for (int64_t i = 2 * int64_t(kPolyWords) * 64 - 1; i >= kDeg; --i) {
    if (!((r[size_t(i) >> 6] >> (i & 63)) & 1u)) continue;
    const int64_t off = i - kDeg;
    const uint64_t* s = t.shifted.data() + size_t(off & 63) * (kPolyWords + 1);
    uint64_t* d = r.data() + (off >> 6);
    const int64_t lim = std::min<int64_t>(kPolyWords + 1, int64_t(r.size()) - (off >> 6));
    for (int64_t w = 0; w < lim; ++w) d[w] ^= s[w];
  }
  r.resize(kPolyWords);
}

inline uint64_t spread32(uint32_t v) {
  uint64_t x = v;
  x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
  x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
  x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}

Poly mulx_mod(const Poly& p) {
  Poly r(kPolyWords, 0);
  for (int w = kPolyWords - 1; w >= 0; --w) r[w] = (p[w] << 1) | (w ? p[w - 1] >> 63 : 0);
  if ((r[kDeg >> 6] >> (kDeg & 63)) & 1u) {
    const Poly& phi = tables().phi;
    for (int w = 0; w < kPolyWords; ++w) r[w] ^= phi[w];
  }
  return r;
}

}  // namespace

const Poly& charpoly() { return tables().phi; }

Poly sqr_mod(const Poly& p) {
  std::vector<uint64_t> r(2 * kPolyWords, 0);
  for (int w = 0; w < kPolyWords; ++w) {
    r[2 * w] = spread32(uint32_t(p[w]));
    r[2 * w + 1] = spread32(uint32_t(p[w] >> 32));
  }
  reduce(r);
  return r;
}

Poly xpow_mod(uint64_t e) {
  Poly r(kPolyWords, 0);
  r[0] = 1;
  for (int b = 63; b >= 0; --b) {
    r = sqr_mod(r);
    if ((e >> b) & 1u) r = mulx_mod(r);
  }
  return r;
}

void jump_window(const uint64_t* win, const Poly& g, uint64_t* out) {
  std::vector<uint64_t> x(kSeqWords);
  raw_sequence(win, x.data(), x.size());
  uint64_t acc[kN] = {0};
  for (int w = 0; w < kPolyWords; ++w) {
    uint64_t bits = g[w];
    while (bits) {
      const int i = w * 64 + __builtin_ctzll(bits);
      bits &= bits - 1;
      const uint64_t* s = x.data() + i;
      for (int j = 0; j < kN; ++j) acc[j] ^= s[j];
    }
  }
  std::memcpy(out, acc, sizeof(acc));
}

std::vector<uint64_t> chunk_windows(uint64_t seed, uint64_t J, uint32_t chunks, int threads) {
  std::vector<uint64_t> out(size_t(std::max<uint32_t>(chunks, 1)) * kN);
  seed_window(seed, out.data());
  if (chunks <= 1) return out;
  uint64_t w1[kN];
  std::memcpy(w1, out.data(), sizeof(w1));
  advance_window(w1);  // W_1: windows reached by jumps are in the image of T
  const Poly step = xpow_mod(J);
  const uint32_t T = uint32_t(std::max(1, std::min<int>(threads, int(chunks - 1))));
  auto work = [&](uint32_t t) {
    const uint32_t c0 = 1 + uint32_t(uint64_t(chunks - 1) * t / T);
    const uint32_t c1 = 1 + uint32_t(uint64_t(chunks - 1) * (t + 1) / T);
    if (c0 >= c1) return;
    jump_window(w1, xpow_mod(uint64_t(c0) * J - 1), out.data() + size_t(c0) * kN);
    for (uint32_t c = c0 + 1; c < c1; ++c)
      jump_window(out.data() + size_t(c - 1) * kN, step, out.data() + size_t(c) * kN);
  };
  std::vector<std::thread> pool;
  for (uint32_t t = 1; t < T; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  return out;
}

uint64_t draw_threshold(double p) {
  if (!(p > 0.0)) return 0;
  const double A = std::ldexp(p, 53);
  if (A >= 9007199254740992.0) return 1ull << 53;
  return uint64_t(std::ceil(A));
}

}  // namespace seraph::mt64
