// Device-side graph construction.
//
//  * dg_rmat / dg_weights: the reference's generate_rmat and assign_weights
//    (ingest.cpp:112-152) bit-for-bit: its sequential std::mt19937_64
//    stream, cut into chunks by GF(2) jump-ahead (mt64.h), one warp per
//    chunk.
//  * dg_symmetrize: symmetrize (graph.cpp:102-118): edge i, then its reverse.
//  * dg_stable_adjacency: the reference's build_csr / build_csc_pages
//    (graph.cpp:30-94) -- a STABLE counting sort by key, so within a source
//    (CSR) or destination (CSC) the input edge order is preserved and the
//    arrays are bit-identical to the reference's.  Chunks of <= 2^30 edges:
//    per-chunk key histograms give the global offsets; each chunk is radix
//    sorted (stable) by key and scattered behind the earlier chunks' edges of
//    the same key.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "devgraph.h"
#include "mt64.h"
#include "errors.h"

namespace seraph {

namespace {

constexpr int kThreads = 256;

inline unsigned grid_of(uint64_t work) {
  const uint64_t g = (work + kThreads - 1) / kThreads;
  return unsigned(std::min<uint64_t>(std::max<uint64_t>(g, 1), 148ull * 32));
}

// ---- std::mt19937_64 on the device (mt64.h) --------------------------------
// The reference's generate_rmat / assign_weights draw from ONE sequential
// std::mt19937_64 stream (ingest.cpp:112-152).  The stream is cut into
// chunks of whole edges; every chunk starts from its own engine window,
// obtained by GF(2) jump-ahead (mt_jump_kernel), and one warp generates it.
namespace mtd {
constexpr int N = mt64::kN, M = mt64::kM;
constexpr int kGenWarps = 8;

__device__ __forceinline__ uint64_t twist(uint64_t xk, uint64_t xk1, uint64_t xm) {
  const uint64_t y = (xk & mt64::kUpper) | (xk1 & mt64::kLower);
  return xm ^ (y >> 1) ^ ((y & 1) ? mt64::kMatrixA : 0ull);
}
__device__ __forceinline__ uint64_t temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  return y ^ (y >> 43);
}
// one twist of a warp's window: nxt = the next 312 raw words after cur
__device__ __forceinline__ void warp_twist(const uint64_t* cur, uint64_t* nxt, int lane) {
  for (int t = lane; t < M; t += 32) nxt[t] = twist(cur[t], cur[t + 1], cur[t + M]);
  __syncwarp();
  for (int t = M + lane; t < N; t += 32)
    nxt[t] = twist(cur[t], t + 1 < N ? cur[t + 1] : nxt[0], nxt[t - M]);
  __syncwarp();
}
}  // namespace mtd

// Jump: out window (dst0 + task) = g(T) window (src0 + task).  The block
// expands its window into the next 20 280 raw words in shared memory (two
// parallel phases per twist), then thread j XORs word i + j over the set
// bits i of g (mt64.h).
__global__ void __launch_bounds__(320) mt_jump_kernel(uint64_t* wins, uint32_t src0, uint32_t dst0,
                                                      const uint64_t* __restrict__ poly) {
  extern __shared__ uint64_t sm[];
  uint64_t* seq = sm;
  uint64_t* g = sm + mt64::kSeqWords;
  const int tid = threadIdx.x;
  const uint64_t* win = wins + size_t(src0 + blockIdx.x) * mtd::N;
  for (int i = tid; i < mtd::N; i += blockDim.x) {
    seq[i] = win[i];
    g[i] = poly[i];
  }
  __syncthreads();
  for (int b = 0; b + 1 < mt64::kSeqWords / mtd::N; ++b) {
    const int k = b * mtd::N + tid;
    if (tid < mtd::M) seq[k + mtd::N] = mtd::twist(seq[k], seq[k + 1], seq[k + mtd::M]);
    __syncthreads();
    if (tid >= mtd::M && tid < mtd::N)
      seq[k + mtd::N] = mtd::twist(seq[k], seq[k + 1], seq[k + mtd::M]);
    __syncthreads();
  }
  if (tid < mtd::N) {
    uint64_t acc = 0;
    for (int w = 0; w < mt64::kPolyWords; ++w) {
      uint64_t bits = g[w];
      while (bits) {
        const int i = w * 64 + __ffsll((long long)bits) - 1;
        bits &= bits - 1;
        acc ^= seq[i + tid];
      }
    }
    wins[size_t(dst0 + blockIdx.x) * mtd::N + tid] = acc;
  }
}

// generate_rmat (ingest.cpp:112-141): chunk ch = edges [ch*per, ch*per+per);
// edge e consumes draws e*scale .. e*scale+scale-1 of the stream, one
// quadrant per draw from the most significant bit down.  Lanes turn the
// warp's 312 fresh draws into 2-bit quadrant codes in a byte ring, then build
// the edges whose draws are all present (consecutive lanes, consecutive edges).
__global__ void __launch_bounds__(256) mt_rmat_kernel(const uint64_t* __restrict__ wins,
                                                      uint32_t chunks, uint64_t per, uint64_t m,
                                                      int scale, uint64_t ta, uint64_t tab,
                                                      uint64_t tabc, uint32_t* __restrict__ src,
                                                      uint32_t* __restrict__ dst) {
  __shared__ uint64_t win[mtd::kGenWarps][2][mtd::N];
  __shared__ uint8_t ring[mtd::kGenWarps][1024];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ch = blockIdx.x * mtd::kGenWarps + warp;
  if (ch >= chunks) return;
  uint64_t e = uint64_t(ch) * per;
  const uint64_t e_end = min(m, e + per);
  uint64_t* cur = win[warp][0];
  uint64_t* nxt = win[warp][1];
  uint8_t* rg = ring[warp];
  for (int i = lane; i < mtd::N; i += 32) cur[i] = wins[size_t(ch) * mtd::N + i];
  __syncwarp();
  uint32_t head = 0, have = 0;
  while (e < e_end) {
    mtd::warp_twist(cur, nxt, lane);
    for (int t = lane; t < mtd::N; t += 32) {
      const uint64_t k = mtd::temper(nxt[t]) >> 11;  // unit_draw = k * 2^-53 (ingest.cpp:21-23)
      rg[(head + have + t) & 1023] = uint8_t((k >= ta) + (k >= tab) + (k >= tabc));
    }
    __syncwarp();
    have += mtd::N;
    const uint64_t left = e_end - e, full = have / uint32_t(scale);
    const uint32_t ne = uint32_t(full < left ? full : left);
    for (uint32_t i = lane; i < ne; i += 32) {
      uint32_t u = 0, v = 0, at = head + i * uint32_t(scale);
      for (int bit = scale - 1; bit >= 0; --bit, ++at) {
        const uint32_t c = rg[at & 1023];  // 0: a, 1: b (dst bit), 2: c (src bit), 3: d (both)
        u |= (c >> 1) << bit;
        v |= (c & 1u) << bit;
      }
      src[e + i] = u;
      dst[e + i] = v;
    }
    __syncwarp();
    e += ne;
    head += ne * uint32_t(scale);
    have -= ne * uint32_t(scale);
    uint64_t* t = cur;
    cur = nxt;
    nxt = t;
  }
}

// assign_weights (ingest.cpp:143-152): w[e] = lo + (draw e) % span.
__global__ void __launch_bounds__(256) mt_weights_kernel(const uint64_t* __restrict__ wins,
                                                         uint32_t chunks, uint64_t per, uint64_t m,
                                                         uint32_t lo, uint64_t span,
                                                         uint32_t* __restrict__ w) {
  __shared__ uint64_t win[mtd::kGenWarps][2][mtd::N];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ch = blockIdx.x * mtd::kGenWarps + warp;
  if (ch >= chunks) return;
  uint64_t e = uint64_t(ch) * per;
  const uint64_t e_end = min(m, e + per);
  uint64_t* cur = win[warp][0];
  uint64_t* nxt = win[warp][1];
  for (int i = lane; i < mtd::N; i += 32) cur[i] = wins[size_t(ch) * mtd::N + i];
  __syncwarp();
  for (; e < e_end; e += mtd::N) {
    mtd::warp_twist(cur, nxt, lane);
    for (int t = lane; t < mtd::N; t += 32)
      if (e + t < e_end) w[e + t] = uint32_t(lo + mtd::temper(nxt[t]) % span);
    __syncwarp();
    uint64_t* t = cur;
    cur = nxt;
    nxt = t;
  }
}

__global__ void symmetrize_kernel(uint64_t m, const uint32_t* __restrict__ src,
                                  const uint32_t* __restrict__ dst, const uint32_t* __restrict__ w,
                                  uint32_t* __restrict__ os, uint32_t* __restrict__ od,
                                  uint32_t* __restrict__ ow) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t u = src[i], v = dst[i];
    reinterpret_cast<uint2*>(os)[i] = make_uint2(u, v);
    reinterpret_cast<uint2*>(od)[i] = make_uint2(v, u);
    if (w) {
      const uint32_t x = w[i];
      reinterpret_cast<uint2*>(ow)[i] = make_uint2(x, x);
    }
  }
}

__global__ void check_ids_kernel(uint32_t n, uint64_t m, const uint32_t* __restrict__ a,
                                 const uint32_t* __restrict__ b, unsigned* bad) {
  bool any = false;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x)
    any |= a[i] >= n || b[i] >= n;
  if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(bad, 1u);
}

// SRPH records (ingest.cpp:153-218): little-endian u32 src, dst[, w] per edge
__global__ void deinterleave_kernel(uint64_t m, const uint32_t* __restrict__ rec, int weighted,
                                    uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                                    uint32_t* __restrict__ w) {
  const uint32_t stride = weighted ? 3 : 2;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t* r = rec + i * stride;
    src[i] = r[0];
    dst[i] = r[1];
    if (weighted) w[i] = r[2];
  }
}

__global__ void check_weights_kernel(uint64_t m, const uint32_t* __restrict__ w, unsigned* bad) {
  bool any = false;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x)
    any |= w[i] < 1u;
  if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(bad, 1u);
}

__global__ void histogram_kernel(uint64_t len, const uint32_t* __restrict__ key, uint32_t* cnt) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < len;
       i += uint64_t(gridDim.x) * blockDim.x)
    atomicAdd(cnt + key[i], 1u);
}

// deg[v] = sum over chunks of cnt[c][v]; deg[n] = 0 (exclusive scan -> offsets)
__global__ void degree_sum_kernel(uint32_t n, uint32_t chunks, const uint32_t* __restrict__ cnt,
                                  unsigned long long* deg) {
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v <= n;
       v += uint64_t(gridDim.x) * blockDim.x) {
    unsigned long long d = 0;
    if (v < n)
      for (uint32_t c = 0; c < chunks; ++c) d += cnt[size_t(c) * n + v];
    deg[v] = d;
  }
}

__global__ void iota_kernel(uint64_t len, uint32_t* p) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < len;
       i += uint64_t(gridDim.x) * blockDim.x)
    p[i] = uint32_t(i);
}

// One sorted chunk: the i-th edge of key v inside the chunk lands behind the
// v-edges of earlier chunks (acc) at its chunk-local rank i - cpref[v].
__global__ void scatter_kernel(uint64_t len, const uint32_t* __restrict__ keys,
                               const uint32_t* __restrict__ idx,
                               const unsigned long long* __restrict__ off,
                               const uint32_t* __restrict__ acc, const uint32_t* __restrict__ cpref,
                               const uint32_t* __restrict__ other, const uint32_t* __restrict__ w,
                               uint32_t* __restrict__ out_other, uint32_t* __restrict__ out_w) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < len;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = keys[i], j = idx[i];
    const unsigned long long pos = off[v] + acc[v] + (i - cpref[v]);
    out_other[pos] = other[j];
    if (w) out_w[pos] = w[j];
  }
}

__global__ void add_counts_kernel(uint32_t n, const uint32_t* __restrict__ cnt, uint32_t* acc) {
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x)
    acc[v] += cnt[v];
}

// Page-local u32 offsets (graph.hpp:49) of every page, packed as
// sr_page_offsets does: page p's range+1 entries start at p*cap + p.
__global__ void page_offsets_kernel(uint32_t n, uint32_t cap, const unsigned long long* __restrict__ off,
                                    uint32_t* local) {
  const uint64_t np = (uint64_t(n) + cap - 1) / cap;
  const uint64_t total = uint64_t(n) + np;
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t p = k / (uint64_t(cap) + 1);
    if (p >= np) p = np - 1;
    const uint64_t i = k - p * (uint64_t(cap) + 1);
    const uint64_t vb = p * cap;
    const uint64_t range = (uint64_t(cap) < n - vb) ? uint64_t(cap) : n - vb;
    if (i <= range) local[k] = uint32_t(off[vb + i] - off[vb]);
  }
}

template <typename T>
struct Tmp {
  T* p = nullptr;
  cudaStream_t s;
  Tmp(size_t count, cudaStream_t st) : s(st) {
    if (count) SR_CUDA(cudaMallocAsync(&p, count * sizeof(T), s));
  }
  ~Tmp() {
    if (p) cudaFreeAsync(p, s);
  }
  Tmp(const Tmp&) = delete;
  Tmp& operator=(const Tmp&) = delete;
};

int key_bits(uint32_t n) {
  int b = 1;
  while (b < 32 && (uint64_t(1) << b) < n) ++b;
  return b;
}

}  // namespace

namespace {

// chunk count of a device stream: one warp per chunk, ~1 K draws minimum
uint32_t mt_chunks(uint64_t units, uint64_t draws_per_unit) {
  uint64_t c = std::max<uint64_t>(1, units * draws_per_unit / 65536);
  c = std::min<uint64_t>(c, 4096);
  if (const char* e = std::getenv("SERAPH_MT_CHUNKS")) c = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));
  return uint32_t(std::min<uint64_t>(c, std::max<uint64_t>(units, 1)));
}

// Engine windows W_{c*J}, c = 0..chunks-1, of std::mt19937_64(seed), on the
// device: W_0 (seeding) and W_1 on the host, W_J = x^{J-1}(T) W_1, then a
// doubling tree of jumps by J*2^r (polynomials x^{J 2^r} mod phi from the host).
void mt_windows(uint64_t seed, uint64_t J, uint32_t chunks, uint64_t* wins, cudaStream_t s) {
  constexpr int N = mt64::kN;
  std::vector<uint64_t> w0(N), w1(N);
  mt64::seed_window(seed, w0.data());
  SR_CUDA(cudaMemcpyAsync(wins, w0.data(), N * 8, cudaMemcpyHostToDevice, s));
  if (chunks > 1) {
    w1 = w0;
    mt64::advance_window(w1.data());
    std::vector<uint64_t> polys;
    const mt64::Poly p0 = mt64::xpow_mod(J - 1);
    polys.insert(polys.end(), p0.begin(), p0.end());
    mt64::Poly q = mt64::xpow_mod(J);
    int rounds = 0;
    for (uint64_t span = 1; span < chunks - 1; span <<= 1, ++rounds) {
      if (rounds) q = mt64::sqr_mod(q);
      polys.insert(polys.end(), q.begin(), q.end());
    }
    Tmp<uint64_t> dpoly(polys.size(), s);
    SR_CUDA(cudaMemcpyAsync(dpoly.p, polys.data(), polys.size() * 8, cudaMemcpyHostToDevice, s));
    SR_CUDA(cudaMemcpyAsync(wins + size_t(chunks) * N, w1.data(), N * 8, cudaMemcpyHostToDevice, s));
    const int smem = int((mt64::kSeqWords + mt64::kPolyWords) * sizeof(uint64_t));
    SR_CUDA(cudaFuncSetAttribute(mt_jump_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    mt_jump_kernel<<<1, 320, smem, s>>>(wins, chunks, 1, dpoly.p);
    SR_CUDA(cudaGetLastError());
    int r = 0;
    for (uint32_t span = 1; span < chunks - 1; span <<= 1, ++r) {
      const uint32_t tasks = std::min(span, chunks - 1 - span);
      mt_jump_kernel<<<tasks, 320, smem, s>>>(wins, 1, 1 + span, dpoly.p + size_t(1 + r) * N);
      SR_CUDA(cudaGetLastError());
    }
    SR_CUDA(cudaStreamSynchronize(s));  // host vectors and dpoly go out of scope
  }
}

}  // namespace

void dg_rmat(int scale, uint64_t m, double a, double b, double c, uint64_t seed, uint32_t* src,
             uint32_t* dst, cudaStream_t s) {
  if (!m) return;
  const double ab = a + b, abc = ab + c;  // ingest.cpp:119-120
  const uint32_t chunks = mt_chunks(m, uint64_t(scale));
  const uint64_t per = (m + chunks - 1) / chunks;
  Tmp<uint64_t> wins(size_t(chunks + 1) * mt64::kN, s);
  mt_windows(seed, per * uint64_t(scale), chunks, wins.p, s);
  mt_rmat_kernel<<<(chunks + mtd::kGenWarps - 1) / mtd::kGenWarps, 256, 0, s>>>(
      wins.p, chunks, per, m, scale, mt64::draw_threshold(a), mt64::draw_threshold(ab),
      mt64::draw_threshold(abc), src, dst);
  SR_CUDA(cudaGetLastError());
}

void dg_weights(uint64_t m, uint64_t seed, uint32_t lo, uint32_t hi, uint32_t* w, cudaStream_t s) {
  if (!m) return;
  const uint32_t chunks = mt_chunks(m, 1);
  const uint64_t per = (m + chunks - 1) / chunks;
  Tmp<uint64_t> wins(size_t(chunks + 1) * mt64::kN, s);
  mt_windows(seed, per, chunks, wins.p, s);
  mt_weights_kernel<<<(chunks + mtd::kGenWarps - 1) / mtd::kGenWarps, 256, 0, s>>>(
      wins.p, chunks, per, m, lo, uint64_t(hi) - lo + 1, w);
  SR_CUDA(cudaGetLastError());
}

void dg_symmetrize(uint64_t m, const uint32_t* src, const uint32_t* dst, const uint32_t* w,
                   uint32_t* os, uint32_t* od, uint32_t* ow, cudaStream_t s) {
  if (!m) return;
  symmetrize_kernel<<<grid_of(m), kThreads, 0, s>>>(m, src, dst, w, os, od, ow);
  SR_CUDA(cudaGetLastError());
}

bool dg_ids_valid(uint32_t n, uint64_t m, const uint32_t* a, const uint32_t* b, cudaStream_t s) {
  if (!m) return true;
  Tmp<unsigned> bad(1, s);
  SR_CUDA(cudaMemsetAsync(bad.p, 0, 4, s));
  check_ids_kernel<<<grid_of(m), kThreads, 0, s>>>(n, m, a, b, bad.p);
  unsigned h = 0;
  SR_CUDA(cudaMemcpyAsync(&h, bad.p, 4, cudaMemcpyDeviceToHost, s));
  SR_CUDA(cudaStreamSynchronize(s));
  return h == 0;
}

void dg_deinterleave(uint64_t m, const uint32_t* records, bool weighted, uint32_t* src,
                     uint32_t* dst, uint32_t* w, cudaStream_t s) {
  if (!m) return;
  deinterleave_kernel<<<grid_of(m), kThreads, 0, s>>>(m, records, weighted ? 1 : 0, src, dst, w);
  SR_CUDA(cudaGetLastError());
}

bool dg_weights_valid(uint64_t m, const uint32_t* w, cudaStream_t s) {
  if (!m || !w) return true;
  Tmp<unsigned> bad(1, s);
  SR_CUDA(cudaMemsetAsync(bad.p, 0, 4, s));
  check_weights_kernel<<<grid_of(m), kThreads, 0, s>>>(m, w, bad.p);
  unsigned h = 0;
  SR_CUDA(cudaMemcpyAsync(&h, bad.p, 4, cudaMemcpyDeviceToHost, s));
  SR_CUDA(cudaStreamSynchronize(s));
  return h == 0;
}

void dg_weights_check_async(uint64_t m, const uint32_t* w, unsigned* bad, cudaStream_t s) {
  if (!m || !w) return;
  check_weights_kernel<<<grid_of(m), kThreads, 0, s>>>(m, w, bad);
  SR_CUDA(cudaGetLastError());
}

void dg_page_offsets(uint32_t n, uint32_t cap, const unsigned long long* off, uint32_t* local,
                     cudaStream_t s) {
  if (!n) return;
  const uint64_t np = (uint64_t(n) + cap - 1) / cap;
  page_offsets_kernel<<<grid_of(n + np), kThreads, 0, s>>>(n, cap, off, local);
  SR_CUDA(cudaGetLastError());
}

void dg_stable_adjacency(uint32_t n, uint64_t m, const uint32_t* key, const uint32_t* other,
                         const uint32_t* w, unsigned long long* out_off, uint32_t* out_other,
                         uint32_t* out_w, cudaStream_t s) {
  uint64_t chunk = uint64_t(1) << 30;  // radix-sort pass size (SERAPH_BUILD_CHUNK: tests)
  if (const char* e = std::getenv("SERAPH_BUILD_CHUNK")) chunk = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));
  const uint64_t C = std::min<uint64_t>(std::max<uint64_t>(m, 1), chunk);
  const uint32_t K = uint32_t((m + C - 1) / C);
  // 1) per-chunk key histograms -> global offsets
  Tmp<uint32_t> cnt(size_t(std::max<uint32_t>(K, 1)) * n, s);
  if (n) SR_CUDA(cudaMemsetAsync(cnt.p, 0, size_t(std::max<uint32_t>(K, 1)) * n * 4, s));
  for (uint32_t c = 0; c < K; ++c) {
    const uint64_t lo = uint64_t(c) * C, len = std::min<uint64_t>(C, m - lo);
    histogram_kernel<<<grid_of(len), kThreads, 0, s>>>(len, key + lo, cnt.p + size_t(c) * n);
  }
  degree_sum_kernel<<<grid_of(uint64_t(n) + 1), kThreads, 0, s>>>(n, K, cnt.p, out_off);
  {
    size_t tb = 0;
    SR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, out_off, out_off, uint64_t(n) + 1, s));
    Tmp<uint8_t> t(tb, s);
    SR_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tb, out_off, out_off, uint64_t(n) + 1, s));
  }
  if (!m || !out_other) return;
  // 2) chunk by chunk: stable radix sort by key, scatter behind earlier chunks
  Tmp<uint32_t> acc(n, s), cpref(n, s);
  SR_CUDA(cudaMemsetAsync(acc.p, 0, size_t(n) * 4, s));
  Tmp<uint32_t> k_out(C, s), i_in(C, s), i_out(C, s);
  size_t sort_bytes = 0, scan_bytes = 0;
  SR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, key, k_out.p, i_in.p, i_out.p, C, 0,
                                          key_bits(n), s));
  SR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, cnt.p, cpref.p, n, s));
  Tmp<uint8_t> tmp(std::max(sort_bytes, scan_bytes), s);
  for (uint32_t c = 0; c < K; ++c) {
    const uint64_t lo = uint64_t(c) * C, len = std::min<uint64_t>(C, m - lo);
    const uint32_t* cc = cnt.p + size_t(c) * n;
    size_t tb = scan_bytes;
    SR_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cc, cpref.p, n, s));
    iota_kernel<<<grid_of(len), kThreads, 0, s>>>(len, i_in.p);
    tb = sort_bytes;
    SR_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key + lo, k_out.p, i_in.p, i_out.p, len, 0,
                                            key_bits(n), s));
    scatter_kernel<<<grid_of(len), kThreads, 0, s>>>(len, k_out.p, i_out.p, out_off, acc.p,
                                                      cpref.p, other + lo, w ? w + lo : nullptr,
                                                      out_other, out_w);
    if (c + 1 < K) add_counts_kernel<<<grid_of(n), kThreads, 0, s>>>(n, cc, acc.p);
  }
  SR_CUDA(cudaGetLastError());
}

}  // namespace seraph
