// Device-side graph construction.
//
//  * dg_rmat / dg_weights: the counter-based RMAT generator and uniform
//    weights of hostgraph.cpp (quadrant law of the reference's generate_rmat,
//    ingest.cpp:112-141; assign_weights range rule, ingest.cpp:143-152) on
//    the GPU, bit-identical to the host version (same splitmix64 stream, same
//    IEEE double comparisons).
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

#include "devgraph.h"
#include "errors.h"

namespace seraph {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

constexpr int kThreads = 256;

inline unsigned grid_of(uint64_t work) {
  const uint64_t g = (work + kThreads - 1) / kThreads;
  return unsigned(std::min<uint64_t>(std::max<uint64_t>(g, 1), 148ull * 32));
}

__global__ void rmat_kernel(int scale, uint64_t m, double a, double ab, double abc, uint64_t seed,
                            uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < m;
       e += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t s = mix64(seed ^ mix64(e));
    uint32_t u = 0, v = 0;
    for (int bit = scale - 1; bit >= 0; --bit) {
      s += 0x9e3779b97f4a7c15ull;
      const double r = double(mix64(s) >> 11) * 0x1.0p-53;
      if (r < a) {
      } else if (r < ab) {
        v |= 1u << bit;
      } else if (r < abc) {
        u |= 1u << bit;
      } else {
        u |= 1u << bit;
        v |= 1u << bit;
      }
    }
    src[e] = u;
    dst[e] = v;
  }
}

__global__ void weights_kernel(uint64_t m, uint64_t seed, uint32_t lo, uint64_t span,
                               uint32_t* __restrict__ w) {
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < m;
       e += uint64_t(gridDim.x) * blockDim.x)
    w[e] = uint32_t(lo + mix64(seed ^ mix64(e + 0x51ull)) % span);
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

void dg_rmat(int scale, uint64_t m, double a, double b, double c, uint64_t seed, uint32_t* src,
             uint32_t* dst, cudaStream_t s) {
  if (!m) return;
  const double ab = a + b, abc = ab + c;
  rmat_kernel<<<grid_of(m), kThreads, 0, s>>>(scale, m, a, ab, abc, seed, src, dst);
  SR_CUDA(cudaGetLastError());
}

void dg_weights(uint64_t m, uint64_t seed, uint32_t lo, uint32_t hi, uint32_t* w, cudaStream_t s) {
  if (!m) return;
  weights_kernel<<<grid_of(m), kThreads, 0, s>>>(m, seed, lo, uint64_t(hi) - lo + 1, w);
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
