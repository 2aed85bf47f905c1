/*
 * seraph_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's algorithms for the hot path, used as
 * the parity checker.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library; the product
 * (libseraph.so) never links or calls it.
 *
 * Parity pinned: the generator and builders are checked bit-for-bit against
 * the reference compiled from /root/reference (oracle/_ref, tests/golden/),
 * the solvers against the reference's golden vectors (test_algorithms.cpp,
 * test_bench.cpp) and reference_solve on the same inputs.
 * PageRank has no reference implementation: "parity unpinned" for it; its
 * conventions are pinned by known-answer tests.
 *
 * Every function cites the reference code it restates.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define UNREACHED 0xffffffffu

/* ---------------------------------------------------------------------- */
/* std::mt19937_64 (the engine behind generate_rmat / assign_weights,
 * ingest.cpp:116, :148).  Standard parameters of the 64-bit Mersenne
 * Twister; restated here because C has no <random>. */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & 0xffffffff80000000ull) | (g->mt[(i + 1) % 312] & 0x7fffffffull);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xb5026f5aa96619e9ull;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71d67fffeda60000ull;
  y ^= (y << 37) & 0xfff7eee000000000ull;
  y ^= y >> 43;
  return y;
}

/* unit_draw (ingest.cpp:18-21): 53-bit uniform double in [0, 1). */
static double unit_draw(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }

/* generate_rmat (ingest.cpp:112-141).  src/dst: 2^scale * edge_factor. */
int oracle_generate_rmat(int scale, uint64_t edge_factor, double a, double b, double c,
                         uint64_t seed, uint32_t* src, uint32_t* dst) {
  if (scale < 1 || scale > 30 || edge_factor < 1) return -1;
  const uint64_t m = ((uint64_t)1 << scale) * edge_factor;
  mt64* g = (mt64*)malloc(sizeof(mt64));
  if (!g) return -2;
  mt64_seed(g, seed);
  const double ab = a + b;
  const double abc = ab + c;
  for (uint64_t e = 0; e < m; ++e) {
    uint32_t s = 0, d = 0;
    for (int bit = scale - 1; bit >= 0; --bit) {
      const double u = unit_draw(g);
      if (u < a) {
      } else if (u < ab) {
        d |= (uint32_t)1 << bit;
      } else if (u < abc) {
        s |= (uint32_t)1 << bit;
      } else {
        s |= (uint32_t)1 << bit;
        d |= (uint32_t)1 << bit;
      }
    }
    src[e] = s;
    dst[e] = d;
  }
  free(g);
  return 0;
}

/* assign_weights (ingest.cpp:143-152): w = lo + rng() % (hi - lo + 1). */
int oracle_assign_weights(uint64_t m, uint64_t seed, uint32_t lo, uint32_t hi, uint32_t* w) {
  if (lo < 1 || lo > hi) return -1;
  mt64* g = (mt64*)malloc(sizeof(mt64));
  if (!g) return -2;
  mt64_seed(g, seed);
  const uint64_t span = (uint64_t)hi - lo + 1;
  for (uint64_t e = 0; e < m; ++e) w[e] = (uint32_t)(lo + mt64_next(g) % span);
  free(g);
  return 0;
}

/* mix64 (bench.cpp:50-55): the bench harness's weight-seed derivation. */
uint64_t oracle_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* symmetrize (graph.cpp:102-118): edge i then its reverse, weights copied. */
void oracle_symmetrize(uint64_t m, const uint32_t* src, const uint32_t* dst, const uint32_t* w,
                       uint32_t* osrc, uint32_t* odst, uint32_t* ow) {
  for (uint64_t i = 0; i < m; ++i) {
    osrc[2 * i] = src[i];
    odst[2 * i] = dst[i];
    osrc[2 * i + 1] = dst[i];
    odst[2 * i + 1] = src[i];
    if (w) {
      ow[2 * i] = w[i];
      ow[2 * i + 1] = w[i];
    }
  }
}

/* Sequential counting sort by key, stable (build_csr graph.cpp:30-48 and the
 * transpose inside build_csc_pages graph.cpp:63-72). */
static void counting_sort(uint32_t n, uint64_t m, const uint32_t* key, const uint32_t* other,
                          const uint32_t* w, uint64_t* off, uint32_t* out_other,
                          uint32_t* out_w) {
  memset(off, 0, sizeof(uint64_t) * ((size_t)n + 1));
  for (uint64_t e = 0; e < m; ++e) off[(size_t)key[e] + 1]++;
  for (size_t v = 1; v <= n; ++v) off[v] += off[v - 1];
  uint64_t* cur = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
  memcpy(cur, off, sizeof(uint64_t) * ((size_t)n + 1));
  for (uint64_t e = 0; e < m; ++e) {
    const uint64_t at = cur[key[e]]++;
    out_other[at] = other[e];
    if (w && out_w) out_w[at] = w[e];
  }
  free(cur);
}

void oracle_build_csr(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                      const uint32_t* w, uint64_t* off, uint32_t* nbr, uint32_t* ow) {
  counting_sort(n, m, src, dst, w, off, nbr, ow);
}

/* build_csc_pages (graph.cpp:50-94): global transpose plus page-local u32
 * offsets; page p's local offsets are local[p*cap + p .. ]. */
void oracle_build_csc(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                      const uint32_t* w, uint32_t cap, uint64_t* in_off, uint32_t* in_src,
                      uint32_t* in_w, uint32_t* local) {
  counting_sort(n, m, dst, src, w, in_off, in_src, in_w);
  const uint64_t np = ((uint64_t)n + cap - 1) / cap;
  for (uint64_t p = 0; p < np; ++p) {
    const uint64_t vb = p * cap;
    const uint64_t ve = vb + cap < n ? vb + cap : n;
    for (uint64_t v = vb; v <= ve; ++v) local[v + p] = (uint32_t)(in_off[v] - in_off[vb]);
  }
}

/* ---------------------------------------------------------------------- */
/* reference_solve (reference.cpp:77-90) */

/* bfs_levels (reference.cpp:13-30): FIFO queue over the CSR. */
void oracle_bfs(uint32_t n, const uint64_t* off, const uint32_t* nbr, uint32_t source,
                uint32_t* depth) {
  for (uint32_t v = 0; v < n; ++v) depth[v] = UNREACHED;
  if (source >= n) return;
  uint32_t* q = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint64_t head = 0, tail = 0;
  depth[source] = 0;
  q[tail++] = source;
  while (head < tail) {
    const uint32_t u = q[head++];
    for (uint64_t k = off[u]; k < off[u + 1]; ++k) {
      const uint32_t v = nbr[k];
      if (depth[v] == UNREACHED) {
        depth[v] = depth[u] + 1;
        q[tail++] = v;
      }
    }
  }
  free(q);
}

/* label_propagation_fixpoint (reference.cpp:32-51): synchronous sweeps. */
void oracle_cc(uint32_t n, const uint64_t* off, const uint32_t* nbr, uint32_t* labels) {
  uint32_t* next = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  for (uint32_t v = 0; v < n; ++v) labels[v] = v;
  int changed = 1;
  while (changed) {
    changed = 0;
    memcpy(next, labels, sizeof(uint32_t) * n);
    for (uint32_t u = 0; u < n; ++u)
      for (uint64_t k = off[u]; k < off[u + 1]; ++k) {
        const uint32_t v = nbr[k];
        if (labels[u] < next[v]) {
          next[v] = labels[u];
          changed = 1;
        }
      }
    memcpy(labels, next, sizeof(uint32_t) * n);
  }
  free(next);
}

/* dijkstra (reference.cpp:53-73): binary min-heap of (dist, vertex),
 * u64 candidate sums, lazy deletion. */
typedef struct {
  uint32_t d, v;
} item;

static int item_less(item a, item b) { return a.d < b.d || (a.d == b.d && a.v < b.v); }

void oracle_sssp(uint32_t n, const uint64_t* off, const uint32_t* nbr, const uint32_t* w,
                 uint32_t source, uint32_t* dist) {
  for (uint32_t v = 0; v < n; ++v) dist[v] = UNREACHED;
  if (source >= n) return;
  size_t cap = 1024, len = 0;
  item* heap = (item*)malloc(sizeof(item) * cap);
  dist[source] = 0;
  heap[len++] = (item){0, source};
  while (len) {
    const item top = heap[0];
    heap[0] = heap[--len];
    for (size_t i = 0;;) { /* sift down */
      size_t l = 2 * i + 1, r = l + 1, s = i;
      if (l < len && item_less(heap[l], heap[s])) s = l;
      if (r < len && item_less(heap[r], heap[s])) s = r;
      if (s == i) break;
      item t = heap[i];
      heap[i] = heap[s];
      heap[s] = t;
      i = s;
    }
    if (top.d != dist[top.v]) continue;
    const uint32_t u = top.v;
    for (uint64_t k = off[u]; k < off[u + 1]; ++k) {
      const uint32_t v = nbr[k];
      const uint64_t cand = (uint64_t)top.d + w[k];
      if (cand < dist[v]) {
        dist[v] = (uint32_t)cand;
        if (len == cap) {
          cap *= 2;
          heap = (item*)realloc(heap, sizeof(item) * cap);
        }
        size_t i = len++;
        heap[i] = (item){dist[v], v};
        while (i > 0) { /* sift up */
          size_t p = (i - 1) / 2;
          if (!item_less(heap[i], heap[p])) break;
          item t = heap[i];
          heap[i] = heap[p];
          heap[p] = t;
          i = p;
        }
      }
    }
  }
  free(heap);
}

/* brute_force_fixpoint (tests/support.hpp:68-97): Bellman-Ford sweeps over
 * the edge list; algo 0 BFS, 1 CC, 2 SSSP. */
void oracle_brute_fixpoint(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                           const uint32_t* w, int algo, uint32_t source, uint32_t* val) {
  for (uint32_t v = 0; v < n; ++v) val[v] = algo == 1 ? v : (v == source ? 0 : UNREACHED);
  int changed = 1;
  while (changed) {
    changed = 0;
    for (uint64_t i = 0; i < m; ++i) {
      if (val[src[i]] == UNREACHED) continue;
      uint64_t cand;
      if (algo == 0) cand = (uint64_t)val[src[i]] + 1;
      else if (algo == 1) cand = val[src[i]];
      else cand = (uint64_t)val[src[i]] + (w ? w[i] : 1);
      if (cand < val[dst[i]]) {
        val[dst[i]] = (uint32_t)cand;
        changed = 1;
      }
    }
  }
}

/* ---------------------------------------------------------------------- */
/* PageRank oracle (no reference implementation; conventions of DESIGN.md
 * §2 / SURVEY §8(c)): rank0 = 1/N, d = damping, `iters` synchronous Jacobi
 * sweeps rank'[v] = (1-d)/N + d * sum_{u->v} rank[u]/outdeg(u), dangling
 * mass dropped, fp64 accumulation, pull over the CSC as in engine.cpp:103-128. */
void oracle_pagerank(uint32_t n, const uint64_t* in_off, const uint32_t* in_src,
                     const uint64_t* out_off, uint32_t iters, double damping, double* rank) {
  double* contrib = (double*)malloc(sizeof(double) * (n ? n : 1));
  const double base = n ? (1.0 - damping) / (double)n : 0.0;
  for (uint32_t v = 0; v < n; ++v) rank[v] = n ? 1.0 / (double)n : 0.0;
  for (uint32_t it = 0; it < iters; ++it) {
    for (uint32_t u = 0; u < n; ++u) {
      const uint64_t d = out_off[u + 1] - out_off[u];
      contrib[u] = d ? rank[u] / (double)d : 0.0;
    }
    for (uint32_t v = 0; v < n; ++v) {
      double s = 0.0;
      for (uint64_t k = in_off[v]; k < in_off[v + 1]; ++k) s += contrib[in_src[k]];
      rank[v] = base + damping * s;
    }
  }
  free(contrib);
}

/* n-th output (1-based) of std::mt19937_64 seeded with `seed`; the C++
 * standard pins the 10000th output of the default seed 5489 at
 * 9981545732273789042 ([rand.predef]). */
uint64_t oracle_mt64_nth(uint64_t seed, uint64_t nth) {
  mt64* g = (mt64*)malloc(sizeof(mt64));
  mt64_seed(g, seed);
  uint64_t x = 0;
  for (uint64_t i = 0; i < nth; ++i) x = mt64_next(g);
  free(g);
  return x;
}
