// ef_bandmerge.cu -- the cross-band seam merge on the device (the union-find
// of trace_edges_parallel, hysteresis.py:104-130, over the bands' edge rows).
//
// Input: nbands blocks of 2*W entries in band order ([0,W) top row, [W,2W)
// bottom row of each band), each a band-LOCAL component id (-1 = background)
// and a strong flag (ef_band_edges' output, all_gathered across ranks).  Every
// rank runs the same merge on the same gathered rows, so every rank reaches
// the same decision with no further exchange.
//
// The union-find runs over entry positions p in [0, n), n = nbands * 2W:
//   K_insert  entries of one band with the same id are one component: a
//             global id (band << 40 | id) is hashed (open addressing, linear
//             probing, atomicCAS on the key) and each slot keeps the smallest
//             position holding that id (atomicMin) as its representative
//   K_unite   every entry is united with its representative, and every bottom
//             entry of band b with the top entries of band b+1 at x-1, x, x+1
//             (8-connectivity across the seam, hysteresis.py:113-125); lock-free
//             union (link the larger root under the smaller one by atomicCAS)
//   K_strong  strong entries mark their root
//   K_out     out[p] = strong flag of p's root (0 for background)
// Four stream-ordered launches; a pass is a few microseconds at C4's 8 bands x
// 32768 entries.  Bit-identical to the host ef_band_merge (ef_abi.cu), which
// the GPU tests compare it with.
#include <cstdint>

#include "ef_internal.h"

namespace ef {

namespace {

constexpr int BM_THREADS = 256;
constexpr unsigned long long kEmptyKey = ~0ull;

__device__ __forceinline__ unsigned long long mix64(unsigned long long k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

// root with path halving; only non-root entries are rewritten (to an
// ancestor), so a concurrent link of a root is never lost
__device__ __forceinline__ int bm_find(int* par, int a) {
    int p = par[a];
    while (p != a) {
        const int gp = par[p];
        if (gp != p) par[a] = gp;
        a = p;
        p = par[a];
    }
    return a;
}

__device__ __forceinline__ int bm_find_ro(const int* __restrict__ par, int a) {
    int p = par[a];
    while (p != a) {
        a = p;
        p = par[a];
    }
    return a;
}

__device__ __forceinline__ void bm_unite(int* par, int a, int b) {
    while (true) {
        a = bm_find(par, a);
        b = bm_find(par, b);
        if (a == b) return;
        if (a > b) {
            const int t = a;
            a = b;
            b = t;
        }
        // link root b under the smaller root a; if b stopped being a root, retry
        if (atomicCAS(&par[b], b, a) == b) return;
    }
}

__global__ void bm_insert_kernel(int n, int W, const int64_t* __restrict__ ids, int* __restrict__ par,
                                 int* __restrict__ hslot, unsigned long long* keys, int* rep, unsigned mask) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int64_t id = ids[p];
    if (id < 0) {
        par[p] = -1;
        return;
    }
    par[p] = p;
    const unsigned long long key = ((unsigned long long)(p / (2 * W)) << 40) | (unsigned long long)id;
    unsigned h = (unsigned)mix64(key) & mask;
    while (true) {
        const unsigned long long old = atomicCAS(&keys[h], kEmptyKey, key);
        if (old == kEmptyKey || old == key) break;
        h = (h + 1) & mask;
    }
    atomicMin(&rep[h], p);
    hslot[p] = (int)h;
}

__global__ void bm_unite_kernel(int n, int W, const int64_t* __restrict__ ids, int* par,
                                const int* __restrict__ hslot, const int* __restrict__ rep) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n || ids[p] < 0) return;
    const int r = rep[hslot[p]];
    if (r != p) bm_unite(par, p, r);
    const int band = p / (2 * W), e = p - band * 2 * W;
    if (e < W || (band + 1) * 2 * W >= n) return;  // not a bottom entry, or the last band
    const int x = e - W;
    const int q0 = (band + 1) * 2 * W;  // top row of the band below
    for (int s = -1; s <= 1; ++s) {
        const int x2 = x + s;
        if (x2 < 0 || x2 >= W || ids[q0 + x2] < 0) continue;
        bm_unite(par, p, q0 + x2);
    }
}

__global__ void bm_strong_kernel(int n, const uint8_t* __restrict__ strong, const int* __restrict__ par,
                                 uint8_t* flag) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n || !strong[p] || par[p] < 0) return;
    flag[bm_find_ro(par, p)] = 1;
}

__global__ void bm_out_kernel(int n, const int* __restrict__ par, const uint8_t* __restrict__ flag,
                              uint8_t* __restrict__ out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    out[p] = par[p] < 0 ? 0 : flag[bm_find_ro(par, p)];
}

unsigned table_size(long long n) {
    unsigned t = 1024;
    while ((long long)t < 2 * n) t <<= 1;
    return t;
}

struct BmLayout {
    size_t par, hslot, flag, keys, rep, total;
    unsigned T;
};

BmLayout bm_layout(int nbands, int W) {
    const long long n = (long long)nbands * 2 * W;
    BmLayout L;
    L.T = table_size(n);
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    L.par = 0;
    L.hslot = al(L.par + sizeof(int) * n);
    L.flag = al(L.hslot + sizeof(int) * n);
    L.keys = al(L.flag + (size_t)n);
    L.rep = al(L.keys + sizeof(unsigned long long) * L.T);
    L.total = al(L.rep + sizeof(int) * L.T);
    return L;
}

}  // namespace

size_t band_merge_scratch_bytes(int nbands, int W) { return bm_layout(nbands, W).total; }

cudaError_t launch_band_merge(int nbands, int W, const int64_t* ids, const uint8_t* strong, uint8_t* out,
                              void* scratch, cudaStream_t st) {
    const BmLayout L = bm_layout(nbands, W);
    const int n = nbands * 2 * W;
    char* s = static_cast<char*>(scratch);
    int* par = reinterpret_cast<int*>(s + L.par);
    int* hslot = reinterpret_cast<int*>(s + L.hslot);
    uint8_t* flag = reinterpret_cast<uint8_t*>(s + L.flag);
    auto* keys = reinterpret_cast<unsigned long long*>(s + L.keys);
    int* rep = reinterpret_cast<int*>(s + L.rep);
    cudaError_t e;
    if ((e = cudaMemsetAsync(flag, 0, (size_t)n, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(keys, 0xff, sizeof(unsigned long long) * L.T, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(rep, 0x7f, sizeof(int) * L.T, st)) != cudaSuccess) return e;  // 0x7f7f7f7f > any p
    const int g = (n + BM_THREADS - 1) / BM_THREADS;
    bm_insert_kernel<<<g, BM_THREADS, 0, st>>>(n, W, ids, par, hslot, keys, rep, L.T - 1);
    bm_unite_kernel<<<g, BM_THREADS, 0, st>>>(n, W, ids, par, hslot, rep);
    bm_strong_kernel<<<g, BM_THREADS, 0, st>>>(n, strong, par, flag);
    bm_out_kernel<<<g, BM_THREADS, 0, st>>>(n, par, flag, out);
    return cudaGetLastError();
}

}  // namespace ef
