/*
 * oracle_par.c -- TEST INFRASTRUCTURE ONLY (part of liboracle.so).
 *
 * Multi-threaded (OpenMP) restatements of the reference's graph pipeline and
 * of the PageRank checker, for the sizes the sequential restatements in
 * seraph_oracle.c cannot reach in a bench run (BASELINE configs C3/C4):
 *
 *  - oracle_generate_rmat_par / oracle_assign_weights_par: generate_rmat and
 *    assign_weights (ingest.cpp:112-152) -- ONE std::mt19937_64 stream --
 *    split into chunks whose engine states are obtained by GF(2) jump-ahead:
 *    the characteristic polynomial phi of MT19937-64 (Berlekamp-Massey on the
 *    output bits), x^J mod phi by square-and-multiply, and the state J steps
 *    ahead as the XOR of the raw words selected by that polynomial (Horner
 *    form of g(T)).  Bit-identical to the sequential stream (tests/test_oracle.py
 *    checks it against oracle_generate_rmat, itself pinned to the reference).
 *  - oracle_symmetrize_par (graph.cpp:102-118), oracle_build_adjacency_par
 *    (build_csr graph.cpp:30-48 with key = src; the CSC of build_csc_pages
 *    graph.cpp:50-94 with key = dst): stable counting sorts, so the arrays
 *    equal the reference's.
 *  - oracle_pagerank_par: the fp64 PageRank checker (pull over the CSC in
 *    the reference's pull_destination structure, engine.cpp:103-128;
 *    out-degree from the CSR offsets, graph.hpp:38-40).  Parity unpinned: the
 *    reference has no PageRank; conventions in DESIGN.md §2.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs load this library.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MT_N 312
#define MT_M 156
#define DEG 19937
#define PW 312             /* words of a residue mod phi (and of phi) */
#define SEQ (MT_N * 65)    /* raw words one jump reads */

static uint64_t mt_twist(uint64_t xk, uint64_t xk1, uint64_t xm) {
  uint64_t y = (xk & 0xffffffff80000000ull) | (xk1 & 0x7fffffffull);
  return xm ^ (y >> 1) ^ ((y & 1) ? 0xb5026f5aa96619e9ull : 0ull);
}

static uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71d67fffeda60000ull;
  y ^= (y << 37) & 0xfff7eee000000000ull;
  return y ^ (y >> 43);
}

/* a generator positioned by its raw-word window (x[k] .. x[k+311]) */
typedef struct {
  uint64_t x[MT_N];
  int idx;
} mtgen;

static uint64_t mtgen_next(mtgen* g) {
  if (g->idx >= MT_N) {
    for (int i = 0; i < MT_N; ++i)
      g->x[i] = mt_twist(g->x[i], g->x[(i + 1) % MT_N], g->x[(i + MT_M) % MT_N]);
    g->idx = 0;
  }
  return mt_temper(g->x[g->idx++]);
}

static void mt_seed_window(uint64_t seed, uint64_t* w) {
  w[0] = seed;
  for (int i = 1; i < MT_N; ++i) w[i] = 6364136223846793005ull * (w[i - 1] ^ (w[i - 1] >> 62)) + (uint64_t)i;
}

static void mt_raw(const uint64_t* win, uint64_t* x, size_t len) {
  memcpy(x, win, MT_N * 8);
  for (size_t k = 0; k + MT_N < len; ++k) x[k + MT_N] = mt_twist(x[k], x[k + 1], x[k + MT_M]);
}

/* ---- phi = characteristic polynomial (Berlekamp-Massey over GF(2)) ---- */
static uint64_t g_phi[PW];
static uint64_t g_phi_sh[64][PW + 1]; /* phi << b */
static int g_phi_ready = 0;

static int getbit(const uint64_t* v, size_t i) { return (int)((v[i >> 6] >> (i & 63)) & 1u); }

static void phi_init(void) {
#pragma omp critical(oracle_phi)
  {
    if (!g_phi_ready) {
      const size_t n2 = 2 * (size_t)DEG, W = n2 / 64 + 4;
      uint64_t* x = (uint64_t*)malloc((n2 + 2 * MT_N) * 8);
      uint64_t win[MT_N];
      mt_seed_window(5489u, win);
      mt_raw(win, x, n2 + 2 * MT_N);
      uint8_t* s = (uint8_t*)malloc(n2);
      for (size_t i = 0; i < n2; ++i) s[i] = (uint8_t)(x[MT_N + i] & 1u);
      uint64_t* Cp = (uint64_t*)calloc(W, 8);
      uint64_t* Bp = (uint64_t*)calloc(W, 8);
      uint64_t* Tp = (uint64_t*)calloc(W, 8);
      Cp[0] = Bp[0] = 1;
      size_t L = 0, m = 1;
      for (size_t n = 0; n < n2; ++n) {
        int d = s[n];
        for (size_t i = 1; i <= L; ++i) d ^= getbit(Cp, i) & s[n - i];
        if (!d) {
          ++m;
          continue;
        }
        const int grow = 2 * L <= n;
        if (grow) memcpy(Tp, Cp, W * 8);
        for (size_t i = 0; i <= n && i + m < W * 64; ++i) /* deg B <= n */
          if (getbit(Bp, i)) Cp[(i + m) >> 6] ^= 1ull << ((i + m) & 63);
        if (grow) {
          L = n + 1 - L;
          memcpy(Bp, Tp, W * 8);
          m = 1;
        } else {
          ++m;
        }
      }
      memset(g_phi, 0, sizeof(g_phi));
      for (size_t k = 0; k <= L && L == DEG; ++k)
        if (getbit(Cp, L - k)) g_phi[k >> 6] |= 1ull << (k & 63);
      for (int b = 0; b < 64; ++b) {
        memset(g_phi_sh[b], 0, sizeof(g_phi_sh[b]));
        for (int w = 0; w < PW; ++w) {
          g_phi_sh[b][w] |= b ? g_phi[w] << b : g_phi[w];
          if (b) g_phi_sh[b][w + 1] |= g_phi[w] >> (64 - b);
        }
      }
      free(x);
      free(s);
      free(Cp);
      free(Bp);
      free(Tp);
      g_phi_ready = 1;
    }
  }
}

/* r (2*PW words) -> r mod phi in r[0..PW) */
static void poly_reduce(uint64_t* r) {
  for (long i = 2L * PW * 64 - 1; i >= DEG; --i) {
    if (!((r[i >> 6] >> (i & 63)) & 1u)) continue;
    const long off = i - DEG, wo = off >> 6;
    const uint64_t* sh = g_phi_sh[off & 63];
    const long lim = (2L * PW - wo) < (PW + 1) ? (2L * PW - wo) : (PW + 1);
    for (long w = 0; w < lim; ++w) r[wo + w] ^= sh[w];
  }
}

static uint64_t spread32(uint32_t v) {
  uint64_t r = 0;
  for (int i = 0; i < 32; ++i) r |= (uint64_t)((v >> i) & 1u) << (2 * i);
  return r;
}

/* out = x^e mod phi */
static void poly_xpow(uint64_t e, uint64_t* out) {
  uint64_t r[2 * PW];
  memset(r, 0, sizeof(r));
  r[0] = 1;
  for (int b = 63; b >= 0; --b) {
    uint64_t sq[2 * PW];
    for (int w = 0; w < PW; ++w) {
      sq[2 * w] = spread32((uint32_t)r[w]);
      sq[2 * w + 1] = spread32((uint32_t)(r[w] >> 32));
    }
    poly_reduce(sq);
    memset(r, 0, sizeof(r));
    memcpy(r, sq, PW * 8);
    if ((e >> b) & 1u) { /* r *= x */
      for (int w = PW - 1; w >= 0; --w) r[w] = (r[w] << 1) | (w ? r[w - 1] >> 63 : 0);
      if ((r[DEG >> 6] >> (DEG & 63)) & 1u)
        for (int w = 0; w < PW; ++w) r[w] ^= g_phi[w];
    }
  }
  memcpy(out, r, PW * 8);
}

/* out = g(T) win: out[j] = XOR_{i : g_i = 1} x[i + j] (win = W_k, k >= 1) */
static void window_jump(const uint64_t* win, const uint64_t* g, uint64_t* out) {
  uint64_t* x = (uint64_t*)malloc(SEQ * 8);
  mt_raw(win, x, SEQ);
  uint64_t acc[MT_N];
  memset(acc, 0, sizeof(acc));
  for (int i = 0; i < DEG; ++i)
    if ((g[i >> 6] >> (i & 63)) & 1u)
      for (int j = 0; j < MT_N; ++j) acc[j] ^= x[i + j];
  memcpy(out, acc, sizeof(acc));
  free(x);
}

/* generator positioned at output index `pos` of std::mt19937_64(seed) */
static void mtgen_at(uint64_t seed, uint64_t pos, mtgen* g) {
  uint64_t w0[MT_N];
  mt_seed_window(seed, w0);
  g->idx = MT_N;
  if (pos == 0) {
    memcpy(g->x, w0, sizeof(w0));
    return;
  }
  uint64_t w1[MT_N], poly[PW];
  memcpy(w1, w0 + 1, (MT_N - 1) * 8);
  w1[MT_N - 1] = mt_twist(w0[0], w0[1], w0[MT_M]); /* W_1 */
  phi_init();
  poly_xpow(pos - 1, poly);
  window_jump(w1, poly, g->x);
}

static int nthreads(int t) { return t > 0 ? t : omp_get_max_threads(); }

/* generate_rmat (ingest.cpp:112-141) on `threads` threads, bit-exact. */
int oracle_generate_rmat_par(int scale, uint64_t edge_factor, double a, double b, double c,
                             uint64_t seed, uint32_t* src, uint32_t* dst, int threads) {
  if (scale < 1 || scale > 30 || edge_factor < 1) return -1;
  const uint64_t m = ((uint64_t)1 << scale) * edge_factor;
  const double ab = a + b, abc = ab + c;
  const int T = nthreads(threads);
  const uint64_t chunks = m < (uint64_t)T * 4 ? m : (uint64_t)T * 4;
  const uint64_t per = (m + chunks - 1) / chunks;
#pragma omp parallel for schedule(dynamic, 1) num_threads(T)
  for (uint64_t ch = 0; ch < chunks; ++ch) {
    mtgen g;
    mtgen_at(seed, ch * per * (uint64_t)scale, &g);
    const uint64_t lo = ch * per, hi = lo + per < m ? lo + per : m;
    for (uint64_t e = lo; e < hi; ++e) {
      uint32_t s = 0, d = 0;
      for (int bit = scale - 1; bit >= 0; --bit) {
        const double u = (double)(mtgen_next(&g) >> 11) * 0x1.0p-53; /* unit_draw */
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
  }
  return 0;
}

/* assign_weights (ingest.cpp:143-152) on `threads` threads, bit-exact. */
int oracle_assign_weights_par(uint64_t m, uint64_t seed, uint32_t lo, uint32_t hi, uint32_t* w,
                              int threads) {
  if (lo < 1 || lo > hi) return -1;
  if (!m) return 0;
  const uint64_t span = (uint64_t)hi - lo + 1;
  const int T = nthreads(threads);
  const uint64_t chunks = m < (uint64_t)T * 4 ? m : (uint64_t)T * 4;
  const uint64_t per = (m + chunks - 1) / chunks;
#pragma omp parallel for schedule(dynamic, 1) num_threads(T)
  for (uint64_t ch = 0; ch < chunks; ++ch) {
    mtgen g;
    mtgen_at(seed, ch * per, &g);
    const uint64_t e0 = ch * per, e1 = e0 + per < m ? e0 + per : m;
    for (uint64_t e = e0; e < e1; ++e) w[e] = (uint32_t)(lo + mtgen_next(&g) % span);
  }
  return 0;
}

/* symmetrize (graph.cpp:102-118): edge i, then its reverse. */
void oracle_symmetrize_par(uint64_t m, const uint32_t* src, const uint32_t* dst,
                           const uint32_t* w, uint32_t* os, uint32_t* od, uint32_t* ow,
                           int threads) {
#pragma omp parallel for schedule(static) num_threads(nthreads(threads))
  for (uint64_t i = 0; i < m; ++i) {
    os[2 * i] = src[i];
    od[2 * i] = dst[i];
    os[2 * i + 1] = dst[i];
    od[2 * i + 1] = src[i];
    if (w) ow[2 * i] = ow[2 * i + 1] = w[i];
  }
}

/* Stable counting sort of edges by key (build_csr graph.cpp:30-48 with
 * key = src / other = dst; the global CSC of build_csc_pages graph.cpp:50-94
 * with key = dst / other = src): off (n+1), out_other, out_w (nullable).
 * Two stable levels: edges scattered into coarse key buckets in
 * (thread, input) order, then every bucket counting-sorted by exact key. */
int oracle_build_adjacency_par(uint32_t n, uint64_t m, const uint32_t* key,
                               const uint32_t* other, const uint32_t* w, uint64_t* off,
                               uint32_t* out_other, uint32_t* out_w, int threads) {
  const int T = nthreads(threads);
  off[0] = 0;
  if (n == 0) return 0;
  const uint64_t bsz = ((uint64_t)n + 1023) / 1024;
  const uint32_t nb = (uint32_t)(((uint64_t)n + bsz - 1) / bsz); /* every bucket non-empty */
  uint64_t* cnt = (uint64_t*)calloc((size_t)T * nb, 8);
  uint32_t* tk = (uint32_t*)malloc((m ? m : 1) * 4);
  uint32_t* to = (uint32_t*)malloc((m ? m : 1) * 4);
  uint32_t* tw = w ? (uint32_t*)malloc((m ? m : 1) * 4) : NULL;
  if (!cnt || !tk || !to || (w && !tw)) return -2;
  int NT = T;
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num(), nt = omp_get_num_threads();
    const uint64_t lo = m * t / nt, hi = m * (t + 1) / nt;
    uint64_t* c = cnt + (size_t)t * nb;
    for (uint64_t e = lo; e < hi; ++e) ++c[key[e] / bsz];
#pragma omp barrier
#pragma omp single
    {
      NT = nt;
      uint64_t run = 0;
      for (uint32_t b = 0; b < nb; ++b)
        for (int u = 0; u < nt; ++u) {
          const uint64_t x = cnt[(size_t)u * nb + b];
          cnt[(size_t)u * nb + b] = run;
          run += x;
        }
    }
    for (uint64_t e = lo; e < hi; ++e) {
      const uint64_t at = c[key[e] / bsz]++;
      tk[at] = key[e];
      to[at] = other[e];
      if (w) tw[at] = w[e];
    }
  }
  /* bucket b now spans [start_b, end_b) in (thread, input) order */
  uint64_t* bstart = (uint64_t*)malloc((nb + 1) * 8);
  {
    /* after the scatter, cnt[(T-1)*nb + b] is the end of bucket b */
    for (uint32_t b = 0; b < nb; ++b) bstart[b + 1] = cnt[(size_t)(NT - 1) * nb + b];
    bstart[0] = 0;
  }
#pragma omp parallel for schedule(dynamic, 1) num_threads(T)
  for (uint32_t b = 0; b < nb; ++b) {
    const uint64_t k0 = (uint64_t)b * bsz, k1 = k0 + bsz < n ? k0 + bsz : n;
    const uint64_t e0 = bstart[b], e1 = bstart[b + 1];
    uint64_t* c = (uint64_t*)calloc(k1 - k0 + 1, 8);
    for (uint64_t e = e0; e < e1; ++e) ++c[tk[e] - k0 + 1];
    for (uint64_t k = 0; k < k1 - k0; ++k) c[k + 1] += c[k];
    for (uint64_t k = 0; k < k1 - k0; ++k) off[k0 + k + 1] = e0 + c[k + 1];
    for (uint64_t e = e0; e < e1; ++e) {
      const uint64_t at = e0 + c[tk[e] - k0]++;
      out_other[at] = to[e];
      if (w) out_w[at] = tw[e];
    }
    free(c);
  }
  free(bstart);
  free(cnt);
  free(tk);
  free(to);
  free(tw);
  return 0;
}

/* PageRank checker, fp64: rank0 = 1/N; 20 synchronous (Jacobi) iterations of
 * rank'(v) = (1-d)/N + d * sum_{u -> v} rank(u)/outdeg(u), dangling mass
 * dropped.  in_off/in_src: global CSC (the pages' in_sources
 * in destination order, engine.cpp:103-128); out_off: CSR offsets
 * (out_degree, graph.hpp:38-40). */
void oracle_pagerank_par(uint32_t n, const uint64_t* in_off, const uint32_t* in_src,
                         const uint64_t* out_off, uint32_t iters, double damping, double* rank,
                         int threads) {
  const int T = nthreads(threads);
  double* contrib = (double*)malloc((n ? n : 1) * 8);
  const double base = (1.0 - damping) / (double)n;
#pragma omp parallel for schedule(static) num_threads(T)
  for (uint32_t v = 0; v < n; ++v) rank[v] = 1.0 / (double)n;
  for (uint32_t it = 0; it < iters; ++it) {
#pragma omp parallel for schedule(static) num_threads(T)
    for (uint32_t u = 0; u < n; ++u) {
      const uint64_t d = out_off[u + 1] - out_off[u];
      contrib[u] = d ? rank[u] / (double)d : 0.0;
    }
#pragma omp parallel for schedule(dynamic, 4096) num_threads(T)
    for (uint32_t v = 0; v < n; ++v) {
      double s = 0.0;
      for (uint64_t k = in_off[v]; k < in_off[v + 1]; ++k) s += contrib[in_src[k]];
      rank[v] = base + damping * s;
    }
  }
  free(contrib);
}

/* max |a-b|, max relative |a-b|/|b| over b > floor, sum |a-b| (PageRank parity report) */
void oracle_pr_compare(uint32_t n, const float* got, const double* want, double rel_floor,
                       double* out3, int threads) {
  double mx = 0, mr = 0, l1 = 0;
#pragma omp parallel for schedule(static) num_threads(nthreads(threads)) reduction(max : mx, mr) reduction(+ : l1)
  for (uint32_t v = 0; v < n; ++v) {
    const double d = fabs((double)got[v] - want[v]);
    if (d > mx) mx = d;
    l1 += d;
    if (want[v] > rel_floor && d / want[v] > mr) mr = d / want[v];
  }
  out3[0] = mx;
  out3[1] = mr;
  out3[2] = l1;
}
