// Host-side graph utilities of libseraph (no GPU needed):
//  * the reference's generate_rmat / assign_weights (ingest.cpp:112-152)
//    bit-for-bit -- its std::mt19937_64 stream cut into chunks by GF(2)
//    jump-ahead (mt64.h) and generated on all host threads;
//  * parallel, stable counting-sort builders producing the reference's CSR
//    (build_csr, graph.cpp:30-48) and CSC page layouts (build_csc_pages,
//    graph.cpp:50-94) bit-for-bit: within a source (CSR) or destination
//    (CSC) the input edge order is preserved;
//  * the edge-balanced shard cut used by the multi-GPU path.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <thread>
#include <vector>

#include "mt64.h"
#include "seraph.h"

namespace mt64 = seraph::mt64;

namespace {

int clamp_threads(int t) {
  if (t <= 0) {
    unsigned h = std::thread::hardware_concurrency();
    t = h ? int(h) : 8;
  }
  return std::max(1, std::min(t, 128));
}

template <typename F>
void run_threads(int t, F&& f) {
  std::vector<std::thread> pool;
  for (int k = 1; k < t; ++k) pool.emplace_back(f, k);
  f(0);
  for (auto& th : pool) th.join();
}

// Stable two-level counting sort of (key, other[, w]) by key.  Level 1
// scatters edges into coarse key buckets in (thread, input) order; level 2
// sorts every bucket by exact key.  Both levels are stable, so the output
// equals the reference's sequential counting sort.
void stable_adjacency(uint32_t n, uint64_t m, const uint32_t* key, const uint32_t* other,
                      const uint32_t* w, uint64_t* out_off, uint32_t* out_other,
                      uint32_t* out_w, int threads) {
  const int T = clamp_threads(threads);
  out_off[0] = 0;
  if (n == 0) return;
  const uint32_t nb = std::min<uint32_t>(n, 4096);
  const uint64_t bsize = (uint64_t(n) + nb - 1) / nb;
  std::vector<uint64_t> cnt(size_t(T) * nb, 0);
  run_threads(T, [&](int t) {
    const uint64_t lo = m * t / T, hi = m * (t + 1) / T;
    uint64_t* c = cnt.data() + size_t(t) * nb;
    for (uint64_t e = lo; e < hi; ++e) ++c[key[e] / bsize];
  });
  std::vector<uint64_t> start(size_t(T) * nb);
  std::vector<uint64_t> bucket_lo(nb + 1);
  uint64_t run = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    bucket_lo[b] = run;
    for (int t = 0; t < T; ++t) {
      start[size_t(t) * nb + b] = run;
      run += cnt[size_t(t) * nb + b];
    }
  }
  bucket_lo[nb] = run;
  std::vector<uint32_t> tk(m), to(m), tw(w ? m : 0);
  run_threads(T, [&](int t) {
    const uint64_t lo = m * t / T, hi = m * (t + 1) / T;
    uint64_t* s = start.data() + size_t(t) * nb;
    for (uint64_t e = lo; e < hi; ++e) {
      const uint64_t at = s[key[e] / bsize]++;
      tk[at] = key[e];
      to[at] = other[e];
      if (w) tw[at] = w[e];
    }
  });
  std::atomic<uint32_t> next{0};
  run_threads(T, [&](int) {
    std::vector<uint64_t> local;
    for (uint32_t b; (b = next.fetch_add(1)) < nb;) {
      const uint64_t v0 = uint64_t(b) * bsize;
      if (v0 >= n) continue;
      const uint64_t v1 = std::min<uint64_t>(v0 + bsize, n);
      local.assign(v1 - v0 + 1, 0);
      for (uint64_t i = bucket_lo[b]; i < bucket_lo[b + 1]; ++i) ++local[tk[i] - v0 + 1];
      for (uint64_t v = 1; v <= v1 - v0; ++v) local[v] += local[v - 1];
      for (uint64_t v = v0; v < v1; ++v) out_off[v + 1] = bucket_lo[b] + local[v - v0 + 1];
      for (uint64_t i = bucket_lo[b]; i < bucket_lo[b + 1]; ++i) {
        const uint64_t at = bucket_lo[b] + local[tk[i] - v0]++;
        out_other[at] = to[i];
        if (w && out_w) out_w[at] = tw[i];
      }
    }
  });
}

}  // namespace

extern "C" {

int sr_rmat_generate(int scale, uint64_t edge_factor, double a, double b, double c, double d,
                     uint64_t seed, uint32_t* src, uint32_t* dst, int threads) {
  if (scale < 1 || scale > 31 || edge_factor < 1 || !src || !dst) return SR_E_CONFIG;
  if (a < 0 || b < 0 || c < 0 || d < 0 || std::abs(a + b + c + d - 1.0) > 1e-9) return SR_E_CONFIG;
  const uint64_t m = (uint64_t(1) << scale) * edge_factor;
  // the reference's sums (ingest.cpp:119-120) as integer draw thresholds
  const double ab = a + b, abc = ab + c;
  const uint64_t ta = mt64::draw_threshold(a), tab = mt64::draw_threshold(ab),
                 tabc = mt64::draw_threshold(abc);
  const int T = clamp_threads(threads);
  const uint32_t chunks = uint32_t(std::min<uint64_t>(m, uint64_t(T) * 4));
  const uint64_t per = (m + chunks - 1) / chunks;  // edges per chunk
  const std::vector<uint64_t> wins = mt64::chunk_windows(seed, per * uint64_t(scale), chunks, T);
  std::atomic<uint32_t> next{0};
  run_threads(T, [&](int) {
    for (uint32_t ch; (ch = next.fetch_add(1)) < chunks;) {
      mt64::Engine g;
      g.load(wins.data() + size_t(ch) * mt64::kN);
      const uint64_t lo = uint64_t(ch) * per, hi = std::min(m, lo + per);
      for (uint64_t e = lo; e < hi; ++e) {
        uint32_t u = 0, v = 0;
        for (int bit = scale - 1; bit >= 0; --bit) {
          const uint64_t k = g() >> 11;  // unit_draw (ingest.cpp:21-23) = k * 2^-53
          if (k < ta) {
          } else if (k < tab) {
            v |= 1u << bit;
          } else if (k < tabc) {
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
  });
  return SR_OK;
}

int sr_weights_generate(uint64_t m, uint64_t seed, uint32_t lo, uint32_t hi, uint32_t* w,
                        int threads) {
  if (lo < 1 || lo > hi || (!w && m)) return SR_E_CONFIG;
  if (!m) return SR_OK;
  const uint64_t span = uint64_t(hi) - lo + 1;
  const int T = clamp_threads(threads);
  const uint32_t chunks = uint32_t(std::min<uint64_t>(m, uint64_t(T) * 4));
  const uint64_t per = (m + chunks - 1) / chunks;
  const std::vector<uint64_t> wins = mt64::chunk_windows(seed, per, chunks, T);
  std::atomic<uint32_t> next{0};
  run_threads(T, [&](int) {
    for (uint32_t ch; (ch = next.fetch_add(1)) < chunks;) {
      mt64::Engine g;
      g.load(wins.data() + size_t(ch) * mt64::kN);
      const uint64_t a = uint64_t(ch) * per, b = std::min(m, a + per);
      for (uint64_t e = a; e < b; ++e) w[e] = uint32_t(lo + g() % span);  // ingest.cpp:150
    }
  });
  return SR_OK;
}

int sr_build_csr(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                 const uint32_t* w, uint64_t* out_offsets, uint32_t* out_neighbors,
                 uint32_t* out_weights, int threads) {
  for (uint64_t e = 0; e < m; ++e)
    if (src[e] >= n || dst[e] >= n) return SR_E_INPUT;
  stable_adjacency(n, m, src, dst, w, out_offsets, out_neighbors, out_weights, threads);
  return SR_OK;
}

int sr_build_csc(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                 const uint32_t* w, uint64_t* in_offsets, uint32_t* in_sources,
                 uint32_t* in_weights, int threads) {
  for (uint64_t e = 0; e < m; ++e)
    if (src[e] >= n || dst[e] >= n) return SR_E_INPUT;
  stable_adjacency(n, m, dst, src, w, in_offsets, in_sources, in_weights, threads);
  return SR_OK;
}

int sr_out_offsets(uint32_t n, uint64_t m, const uint32_t* src, uint64_t* out_offsets,
                   int threads) {
  // out-degree prefix only (the push adjacency can be derived on the device)
  const int T = clamp_threads(threads);
  std::vector<std::atomic<uint64_t>> deg(size_t(n) + 1);
  for (auto& d : deg) d.store(0, std::memory_order_relaxed);
  std::atomic<bool> bad{false};
  run_threads(T, [&](int t) {
    const uint64_t lo = m * t / T, hi = m * (t + 1) / T;
    for (uint64_t e = lo; e < hi; ++e) {
      if (src[e] >= n) {
        bad = true;
        return;
      }
      deg[size_t(src[e]) + 1].fetch_add(1, std::memory_order_relaxed);
    }
  });
  if (bad) return SR_E_INPUT;
  out_offsets[0] = 0;
  for (size_t v = 1; v <= n; ++v) out_offsets[v] = out_offsets[v - 1] + deg[v].load();
  return SR_OK;
}

int sr_symmetrize(uint64_t m, const uint32_t* src, const uint32_t* dst, const uint32_t* w,
                  uint32_t* osrc, uint32_t* odst, uint32_t* ow, int threads) {
  // symmetrize (graph.cpp:102-118): edge i then its reverse, weights copied
  const int T = clamp_threads(threads);
  run_threads(T, [&](int t) {
    const uint64_t lo = m * t / T, hi = m * (t + 1) / T;
    for (uint64_t i = lo; i < hi; ++i) {
      osrc[2 * i] = src[i];
      odst[2 * i] = dst[i];
      osrc[2 * i + 1] = dst[i];
      odst[2 * i + 1] = src[i];
      if (w) ow[2 * i] = ow[2 * i + 1] = w[i];
    }
  });
  return SR_OK;
}

int sr_page_offsets(uint32_t n, uint32_t cap, const uint64_t* in_off, uint32_t* local) {
  if (cap < 1) return SR_E_CONFIG;
  const uint64_t np = (uint64_t(n) + cap - 1) / cap;
  for (uint64_t p = 0; p < np; ++p) {
    const uint64_t vb = p * cap, ve = std::min<uint64_t>(vb + cap, n);
    if (in_off[ve] - in_off[vb] > 0xffffffffull) return SR_E_CONFIG;
    uint32_t* out = local + vb + p;
    const uint64_t base = in_off[vb];
    for (uint64_t v = vb; v <= ve; ++v) out[v - vb] = uint32_t(in_off[v] - base);
  }
  return SR_OK;
}

int sr_shard_plan(uint32_t n, const uint64_t* in_off, uint32_t parts, uint32_t* cuts) {
  if (parts < 1 || !cuts) return SR_E_CONFIG;
  const uint64_t m = in_off[n];
  cuts[0] = 0;
  for (uint32_t r = 1; r < parts; ++r) {
    const uint64_t target = m * r / parts;
    const uint64_t* it = std::lower_bound(in_off, in_off + n + 1, target);
    cuts[r] = std::max(cuts[r - 1], uint32_t(std::min<uint64_t>(it - in_off, n)));
  }
  cuts[parts] = n;
  return SR_OK;
}

}  // extern "C"
