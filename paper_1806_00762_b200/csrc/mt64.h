// std::mt19937_64 -- the engine behind the reference's generate_rmat and
// assign_weights (ingest.cpp:112-152) -- with GF(2) jump-ahead, so the
// reference's exact random stream can be cut into independent chunks and
// generated in parallel (host threads, or one warp per chunk on the GPU).
//
// Model.  The raw words satisfy x[k+312] = x[k+156] ^ A(upper33(x[k]) |
// lower31(x[k+1])) (the twist), outputs are temper(x[312+j]).  A "window"
// W_k = (x[k] .. x[k+311]) is exactly the array a freshly twisted
// std::mt19937_64 holds, so an engine loaded with W_k and index 312 emits
// outputs k, k+1, ... .  Window advance is a linear map T on GF(2)^19968
// whose minimal polynomial on windows with k >= 1 is the degree-19937
// characteristic polynomial phi of MT19937-64 (obtained here by
// Berlekamp-Massey from the output bits), hence for k >= 1
//     W_{k+J} = g(T) W_k,  g = x^J mod phi,
// i.e. W_{k+J}[j] = XOR over set bits i of g of x[k+i+j]  (a correlation of
// g with the next 20248 raw words).
#pragma once

#include <cstdint>
#include <vector>

namespace seraph::mt64 {

constexpr int kN = 312;            // state words
constexpr int kM = 156;            // twist offset
constexpr int kDeg = 19937;        // degree of phi
constexpr int kPolyWords = 312;    // residues mod phi (< 19937 bits) and phi itself (19938 bits)
constexpr int kSeqWords = kN * 65; // raw words a jump correlates over (>= 19936 + 312)
constexpr uint64_t kMatrixA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull;
constexpr uint64_t kLower = 0x000000007FFFFFFFull;

using Poly = std::vector<uint64_t>;  // kPolyWords words, bit i = coefficient of x^i

inline uint64_t twist(uint64_t xk, uint64_t xk1, uint64_t xm) {
  const uint64_t y = (xk & kUpper) | (xk1 & kLower);
  return xm ^ (y >> 1) ^ ((y & 1) ? kMatrixA : 0ull);
}

inline uint64_t temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

// W_0: the seeded state (std::mersenne_twister_engine::seed).
void seed_window(uint64_t seed, uint64_t* win);
// W_k -> W_{k+1} in place.
void advance_window(uint64_t* win);
// phi (computed once per process, thread-safe).
const Poly& charpoly();
// x^e mod phi.
Poly xpow_mod(uint64_t e);
// p^2 mod phi.
Poly sqr_mod(const Poly& p);
// out = g(T) win  (win must be a window W_k with k >= 1).
void jump_window(const uint64_t* win, const Poly& g, uint64_t* out);

// std::mt19937_64 loaded from a window: emits outputs k, k+1, ... of W_k.
struct Engine {
  uint64_t mt[kN];
  int idx = kN;
  void load(const uint64_t* win);
  uint64_t operator()();
};

// Windows W_{c*J} for chunks c = 0..chunks-1 of a stream seeded with `seed`
// (chunk 0 = the seeded window), computed on `threads` host threads.
std::vector<uint64_t> chunk_windows(uint64_t seed, uint64_t J, uint32_t chunks, int threads);

// Quadrant thresholds of generate_rmat (ingest.cpp:119-120, 126-136) as
// integers on the 53-bit draw k = x >> 11: (k * 2^-53 < p) <=> (k < T(p)).
uint64_t draw_threshold(double p);

}  // namespace seraph::mt64
