// layout.cuh -- record block of the .lrcvt layout (reference
// lrcvt/layout.py:123-200, build_and_write): in-band voxels ordered by
// (component, region, voxel) -- region = site_of, unassigned voxels keyed
// 0xFFFFFFFF so they close their component's range -- and packed as
// little-endian records {u32 x, y, z; f32 field[m]}.
//
// The order is one stable radix sort of a 64-bit (component << 32 | region)
// key over the in-band voxels listed in increasing order (== np.lexsort((voxel,
// region, component))). Packing writes the record block as a stream of 32-bit
// words, one thread per word, so the stores are fully coalesced.
#pragma once

#include <cstdint>

namespace lrcvt {

constexpr unsigned kUnassignedRegion = 0xFFFFFFFFu;

// key = component << rbits | region code; code = site, or n_sites for an
// unassigned voxel (so it closes its component's range like 0xFFFFFFFF does);
// 32-bit keys whenever the two fields fit. A site id >= n_sites sets *bad.
template <typename K>
__global__ void k_layout_keys(const int* __restrict__ list, int64_t n, const int* __restrict__ comp,
                              const int* __restrict__ site_of, int n_sites, int rbits, K* __restrict__ key,
                              int* __restrict__ bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int v = list[i];
    int s = site_of[v];
    if (s >= n_sites) { atomicExch(bad, 1); s = n_sites; }
    const unsigned code = s >= 0 ? (unsigned)s : (unsigned)n_sites;
    key[i] = ((K)(unsigned)comp[v] << rbits) | (K)code;
  }
}

struct FieldPtrs {
  const float* f[16];
};

// word w of the record block: record i = w / (3 + m), slot j = w % (3 + m)
__global__ void k_layout_pack(const int* __restrict__ vox, int64_t r, int m, int nx, int ny, FieldPtrs fp,
                              unsigned* __restrict__ out) {
  const int words = 3 + m;
  const int64_t total = r * words;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total; w += stride) {
    const int64_t i = w / words;
    const int j = (int)(w - i * words);
    const int v = __ldg(vox + i);
    unsigned word;
    if (j == 0) word = (unsigned)(v % nx);
    else if (j == 1) word = (unsigned)((v / nx) % ny);
    else if (j == 2) word = (unsigned)(v / (nx * ny));
    else word = __float_as_uint(__ldg(fp.f[j - 3] + v));
    __stcs(out + w, word);
  }
}

// region key per record (the reference's u32 key: site or 0xFFFFFFFF), and
// each component's [first, first + count) range
template <typename K>
__global__ void k_layout_index(const K* __restrict__ key, int64_t r, int rbits, int n_sites,
                               unsigned* __restrict__ region_key, int n_comp,
                               long long* __restrict__ comp_first, long long* __restrict__ comp_count) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const K rmask = ((K)1 << rbits) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r; i += stride) {
    const K k = key[i];
    const unsigned code = (unsigned)(k & rmask);
    region_key[i] = code == (unsigned)n_sites ? kUnassignedRegion : code;
    const unsigned c = (unsigned)(k >> rbits);
    if (c >= (unsigned)n_comp) continue;
    if (i == 0 || (unsigned)(key[i - 1] >> rbits) != c) comp_first[c] = i;
    if (i == r - 1 || (unsigned)(key[i + 1] >> rbits) != c) comp_count[c] = i + 1;  // end; count fixed below
  }
}

__global__ void k_layout_counts(int n_comp, const long long* __restrict__ first, long long* __restrict__ count) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n_comp && count[c] > 0) count[c] -= first[c];
}

}  // namespace lrcvt
