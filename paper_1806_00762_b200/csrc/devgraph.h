// Device-side graph construction (devgraph.cu): RMAT/weights generation,
// symmetrize and the reference's stable CSR/CSC builders on the GPU.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace seraph {

// generate_rmat quadrant law on the splitmix64 counter stream (bit-identical
// to sr_rmat_generate); m = 2^scale * edge_factor edges.
void dg_rmat(int scale, uint64_t m, double a, double b, double c, uint64_t seed, uint32_t* src,
             uint32_t* dst, cudaStream_t s);
// uniform [lo, hi] weights (bit-identical to sr_weights_generate)
void dg_weights(uint64_t m, uint64_t seed, uint32_t lo, uint32_t hi, uint32_t* w, cudaStream_t s);
// symmetrize (graph.cpp:102-118): 2m outputs, edge i then (dst, src)
void dg_symmetrize(uint64_t m, const uint32_t* src, const uint32_t* dst, const uint32_t* w,
                   uint32_t* os, uint32_t* od, uint32_t* ow, cudaStream_t s);
// true when every id of a[0..m) and b[0..m) is < n (synchronises s)
bool dg_ids_valid(uint32_t n, uint64_t m, const uint32_t* a, const uint32_t* b, cudaStream_t s);
// Stable counting sort by key (build_csr with key=src, build_csc with
// key=dst): out_off (n+1, u64), out_other/out_w (m; out_other may be null
// for offsets only, out_w null when unweighted).
void dg_stable_adjacency(uint32_t n, uint64_t m, const uint32_t* key, const uint32_t* other,
                         const uint32_t* w, unsigned long long* out_off, uint32_t* out_other,
                         uint32_t* out_w, cudaStream_t s);
// SRPH edge records (src, dst[, w] u32 each) -> separate arrays
void dg_deinterleave(uint64_t m, const uint32_t* records, bool weighted, uint32_t* src,
                     uint32_t* dst, uint32_t* w, cudaStream_t s);
// true when every weight is >= 1 (EdgeList::validate, graph.cpp:9-22; synchronises s)
bool dg_weights_valid(uint64_t m, const uint32_t* w, cudaStream_t s);
// ORs 1 into *bad (device word) when any of the m weights is < 1; no sync.
void dg_weights_check_async(uint64_t m, const uint32_t* w, unsigned* bad, cudaStream_t s);
// page-local u32 offsets of pages of `cap` vertices (layout of sr_page_offsets)
void dg_page_offsets(uint32_t n, uint32_t cap, const unsigned long long* off, uint32_t* local,
                     cudaStream_t s);

}  // namespace seraph
