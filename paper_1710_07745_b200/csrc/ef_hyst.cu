// ef_hyst.cu -- hysteresis edge tracking (trace_edges, hysteresis.py:63-69).
//
// The reference labels 8-connected components of labels != 0 with
// scipy.ndimage.label and keeps those that contain a strong pixel.  The result
// is a set, so any correct connected-component algorithm is bit-exact.  Here:
//
//  H1 hyst_local   one CTA per 64x64 tile: lock-free union-find in shared
//                  memory over the tile's pixels.  Components that do not touch
//                  the tile border are final right away (kept iff they hold a
//                  strong pixel).  Border-touching components become global
//                  nodes, numbered tile*256 + (smallest perimeter slot).
//  H2 hyst_merge   unions nodes across tile seams (right, bottom, and the two
//                  diagonal corners) with an atomicCAS union-find in HBM.
//  H3 hyst_resolve propagates "holds a strong pixel" to every node's root.
//  H4 hyst_final   re-runs the tile CCL only for tiles with undecided
//                  border components and reads their roots' strong flag.
//
// HBM traffic: labels read once (twice for the few pending tiles), final
// written once, plus 9 bytes per perimeter slot (~0.5 B/pixel worst case).
// The same machinery runs per row band for the multi-GPU partition
// (trace_edges_parallel, hysteresis.py:90-131): band-edge components stay
// pending until the cross-band merge.
#include "ef_common.cuh"
#include "ef_internal.h"

namespace ef {

constexpr int HT = 64;          // tile edge
constexpr int HP = 4 * HT;      // perimeter slots per tile
constexpr int H_THREADS = 256;  // 16 pixels per thread
constexpr int NO_POS = 0x7fffffff;

struct TileCCL {
    int par[HT * HT];
    int minpos[HT * HT];
    uint8_t lab[HT * HT];
    uint8_t sflag[HT * HT];
    int pending;
    int nodes;
};

__device__ __forceinline__ int sfind(int* par, int i) {
    while (true) {
        int p = par[i];
        if (p == i) return i;
        int gp = par[p];
        if (gp != p) par[i] = gp;  // path halving: only ever points further up
        i = p;
    }
}

__device__ __forceinline__ void sunite(int* par, int a, int b) {
    while (true) {
        a = sfind(par, a);
        b = sfind(par, b);
        if (a == b) return;
        if (a < b) { int t = a; a = b; b = t; }
        if (atomicCAS(&par[a], a, b) == a) return;
    }
}

__device__ __forceinline__ int gfind(int* par, int i) {
    while (true) {
        int p = par[i];
        if (p == i) return i;
        int gp = par[p];
        if (gp != p) par[i] = gp;
        i = p;
    }
}

__device__ __forceinline__ int gfind_ro(const int* par, int i) {
    while (true) {
        int p = par[i];
        if (p == i) return i;
        i = p;
    }
}

__device__ __forceinline__ void gunite(int* par, int a, int b) {
    while (true) {
        a = gfind(par, a);
        b = gfind(par, b);
        if (a == b) return;
        if (a < b) { int t = a; a = b; b = t; }
        if (atomicCAS(&par[a], a, b) == a) return;
    }
}

struct TileGeo {
    int f, tyi, txi, y0, x0, vh, vw;
};

__device__ __forceinline__ TileGeo tile_geo(long long tile, int H, int W, int tiles_x, int tiles_y) {
    TileGeo g;
    long long per = (long long)tiles_x * tiles_y;
    g.f = (int)(tile / per);
    int t2 = (int)(tile - (long long)g.f * per);
    g.tyi = t2 / tiles_x;
    g.txi = t2 - g.tyi * tiles_x;
    g.y0 = g.tyi * HT;
    g.x0 = g.txi * HT;
    g.vh = min(HT, H - g.y0);
    g.vw = min(HT, W - g.x0);
    return g;
}

// Perimeter slot(s) of tile-local pixel (y, x) given the valid extent; returns
// the smallest slot or NO_POS.  Slots: top row x, bottom row 64+x, left col
// 128+y, right col 192+y.
__device__ __forceinline__ int perim_slot(int y, int x, int vh, int vw) {
    int s = NO_POS;
    if (x == vw - 1) s = 192 + y;
    if (x == 0) s = 128 + y;
    if (y == vh - 1) s = 64 + x;
    if (y == 0) s = x;
    return s;
}

__device__ __forceinline__ void slot_pixel(int s, int vh, int vw, int& y, int& x) {
    if (s < 64) { y = 0; x = s; }
    else if (s < 128) { y = vh - 1; x = s - 64; }
    else if (s < 192) { y = s - 128; x = 0; }
    else { y = s - 192; x = vw - 1; }
}

// Shared tile CCL used by H1 and H4.  After return (and a barrier) par[] holds
// roots for every foreground pixel, sflag[root] marks strong components and
// minpos[root] the smallest perimeter slot (NO_POS if interior).
__device__ void tile_ccl(const uint8_t* __restrict__ labels, int H, int W, const TileGeo& g,
                         TileCCL& s) {
    const int tid = threadIdx.x;
    const int row = tid >> 2, seg = (tid & 3) * 16;
    const uint8_t* frame = labels + (size_t)g.f * H * W;
    const int Y = g.y0 + row;
    uint8_t v[16];
    const uint8_t* src = frame + (size_t)Y * W + g.x0 + seg;
    if (row < g.vh && seg + 16 <= g.vw && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
        uint4 q = *reinterpret_cast<const uint4*>(src);
        const uint8_t* qb = reinterpret_cast<const uint8_t*>(&q);
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = qb[k];
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            int X = seg + k;
            v[k] = (row < g.vh && X < g.vw) ? frame[(size_t)Y * W + g.x0 + X] : 0;
        }
    }
    int run = -1;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        int i = row * HT + seg + k;
        s.lab[i] = v[k];
        s.sflag[i] = 0;
        s.minpos[i] = NO_POS;
        if (v[k]) {
            if (run < 0) run = i;
            s.par[i] = run;  // pre-link runs inside this thread's segment
        } else {
            run = -1;
            s.par[i] = i;
        }
    }
    __syncthreads();
    // unions with W (across segments only), NW, N, NE
#pragma unroll 1
    for (int k = 0; k < 16; ++k) {
        int x = seg + k, i = row * HT + x;
        if (!v[k]) continue;
        if (k == 0 && x > 0 && s.lab[i - 1]) sunite(s.par, i, i - 1);
        if (row > 0) {
            int up = i - HT;
            if (s.lab[up]) sunite(s.par, i, up);
            else {
                if (x > 0 && s.lab[up - 1]) sunite(s.par, i, up - 1);
                if (x < HT - 1 && s.lab[up + 1]) sunite(s.par, i, up + 1);
            }
        }
    }
    __syncthreads();
    // roots, strong flags, perimeter minima.  Roots go to registers first:
    // concurrent path-halving writes could otherwise overwrite a stored root
    // with a non-root ancestor; the forest is only rewritten after a barrier.
    int roots[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        int x = seg + k, i = row * HT + x;
        roots[k] = v[k] ? sfind(s.par, i) : -1;
        if (!v[k]) continue;
        if (v[k] == kStrong) s.sflag[roots[k]] = 1;
        int p = perim_slot(row, x, g.vh, g.vw);
        if (p != NO_POS) atomicMin(&s.minpos[roots[k]], p);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k)
        if (v[k]) s.par[row * HT + seg + k] = roots[k];
    __syncthreads();
}

__global__ void __launch_bounds__(H_THREADS)
hyst_local_kernel(const uint8_t* __restrict__ labels, int H, int W, int tiles_x, int tiles_y,
                  uint8_t* __restrict__ final_out, int* __restrict__ perim, int* __restrict__ gpar,
                  uint8_t* __restrict__ gstrong, uint8_t* __restrict__ pending, WsHeader* hdr) {
    __shared__ TileCCL s;
    const long long tile = blockIdx.x;
    TileGeo g = tile_geo(tile, H, W, tiles_x, tiles_y);
    if (threadIdx.x == 0) { s.pending = 0; s.nodes = 0; }
    tile_ccl(labels, H, W, g, s);
    const int tid = threadIdx.x;
    const int row = tid >> 2, seg = (tid & 3) * 16;
    uint8_t* frame = final_out + (size_t)g.f * H * W;
    bool pend = false;
    if (row < g.vh) {
        alignas(16) uint8_t o[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            int i = row * HT + seg + k;
            uint8_t out = 0;
            if (s.lab[i]) {
                int root = s.par[i];
                if (s.sflag[root]) out = 1;
                else if (s.minpos[root] != NO_POS) pend = true;
            }
            o[k] = out;
        }
        const int Y = g.y0 + row;
        uint8_t* dst = frame + (size_t)Y * W + g.x0 + seg;
        if (seg + 16 <= g.vw && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
            *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(o);
        } else {
            for (int k = 0; k < 16; ++k)
                if (seg + k < g.vw) frame[(size_t)Y * W + g.x0 + seg + k] = o[k];
        }
    }
    if (pend) s.pending = 1;
    // perimeter slots: node id of the component at each slot, -1 if background
    {
        int p = tid;  // H_THREADS == HP
        int y, x;
        slot_pixel(p, g.vh, g.vw, y, x);
        int node = -1;
        bool valid = (p < 64 || (p >= 64 && p < 128)) ? (x < g.vw) : (y < g.vh);
        if (valid) {
            int i = y * HT + x;
            if (s.lab[i]) {
                int root = s.par[i];
                node = (int)(tile * HP) + s.minpos[root];
                if (s.minpos[root] == p) {
                    gpar[node] = node;
                    gstrong[node] = s.sflag[root];
                    atomicAdd(&s.nodes, 1);
                }
            }
        }
        perim[tile * HP + p] = node;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        pending[tile] = (uint8_t)s.pending;
        if (s.nodes) atomicAdd((unsigned long long*)&hdr->stats.border_nodes, (unsigned long long)s.nodes);
        if (s.pending) atomicAdd((unsigned long long*)&hdr->stats.pending_tiles, 1ull);
    }
}

// H2: unions across tile seams.  128 threads per tile: 0..63 right seam rows,
// 64..127 bottom seam columns; thread 0 also does the two corner diagonals.
__global__ void __launch_bounds__(128)
hyst_merge_kernel(int H, int W, int tiles_x, int tiles_y, const int* __restrict__ perim, int* gpar) {
    const long long tile = blockIdx.x;
    TileGeo g = tile_geo(tile, H, W, tiles_x, tiles_y);
    const int t = threadIdx.x;
    const int* pa = perim + tile * HP;
    if (t < 64) {
        if (g.txi + 1 < tiles_x && t < g.vh) {
            int a = pa[192 + t];
            if (a >= 0) {
                const int* pb = perim + (tile + 1) * HP;
                for (int dy = -1; dy <= 1; ++dy) {
                    int y2 = t + dy;
                    if (y2 < 0 || y2 >= g.vh) continue;
                    int b = pb[128 + y2];
                    if (b >= 0) gunite(gpar, a, b);
                }
            }
        }
    } else {
        int x = t - 64;
        if (g.tyi + 1 < tiles_y && x < g.vw) {
            int a = pa[64 + x];
            if (a >= 0) {
                const int* pc = perim + (tile + tiles_x) * HP;
                TileGeo gc = tile_geo(tile + tiles_x, H, W, tiles_x, tiles_y);
                for (int dx = -1; dx <= 1; ++dx) {
                    int x2 = x + dx;
                    if (x2 < 0 || x2 >= gc.vw) continue;
                    int c = pc[x2];
                    if (c >= 0) gunite(gpar, a, c);
                }
            }
        }
    }
    if (t == 0 && g.tyi + 1 < tiles_y) {
        if (g.txi + 1 < tiles_x && g.vw == HT) {  // bottom-right corner -> tile below-right (0,0)
            int a = pa[64 + HT - 1];
            int d = perim[(tile + tiles_x + 1) * HP + 0];
            if (a >= 0 && d >= 0) gunite(gpar, a, d);
        }
        if (g.txi > 0) {  // bottom-left corner -> tile below-left (0, 63)
            int a = pa[64 + 0];
            int d = perim[(tile + tiles_x - 1) * HP + HT - 1];
            if (a >= 0 && d >= 0) gunite(gpar, a, d);
        }
    }
}

// H3: strong flag of every node onto its root.
__global__ void hyst_resolve_kernel(long long nslots, const int* __restrict__ perim, int* gpar,
                                    uint8_t* gstrong) {
    for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < nslots;
         s += (long long)gridDim.x * blockDim.x) {
        int n = perim[s];
        if (n != (int)s) continue;  // the node's own (smallest) slot only
        int r = gfind(gpar, n);
        if (gstrong[n] && r != n) gstrong[r] = 1;
    }
}

// H4: finalise tiles that had undecided border components.
__global__ void __launch_bounds__(H_THREADS)
hyst_final_kernel(const uint8_t* __restrict__ labels, int H, int W, int tiles_x, int tiles_y,
                  uint8_t* __restrict__ final_out, const int* __restrict__ gpar,
                  const uint8_t* __restrict__ gstrong, const uint8_t* __restrict__ pending) {
    __shared__ TileCCL s;
    const long long tile = blockIdx.x;
    if (!pending[tile]) return;
    TileGeo g = tile_geo(tile, H, W, tiles_x, tiles_y);
    tile_ccl(labels, H, W, g, s);
    const int tid = threadIdx.x;
    const int row = tid >> 2, seg = (tid & 3) * 16;
    if (row >= g.vh) return;
    uint8_t* frame = final_out + (size_t)g.f * H * W;
    const int Y = g.y0 + row;
    for (int k = 0; k < 16; ++k) {
        int x = seg + k;
        if (x >= g.vw) break;
        int i = row * HT + x;
        if (!s.lab[i]) continue;
        int root = s.par[i];
        if (s.sflag[root] || s.minpos[root] == NO_POS) continue;
        int node = (int)(tile * HP) + s.minpos[root];
        if (gstrong[gfind_ro(gpar, node)]) frame[(size_t)Y * W + g.x0 + x] = 1;
    }
}

// Band edge export: component root id and strong flag for the top and bottom
// rows of a band (the frame of `rows` rows).
__global__ void band_edges_kernel(int rows, int W, int tiles_x, int tiles_y, const int* __restrict__ perim,
                                  const int* __restrict__ gpar, const uint8_t* __restrict__ gstrong,
                                  int64_t* ids, uint8_t* strong) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * W) return;
    bool bottom = t >= W;
    int x = bottom ? t - W : t;
    long long tile = (long long)(bottom ? tiles_y - 1 : 0) * tiles_x + x / HT;
    int slot = (bottom ? 64 : 0) + x % HT;
    int node = perim[tile * HP + slot];
    if (node < 0) { ids[t] = -1; strong[t] = 0; return; }
    int r = gfind_ro(gpar, node);
    ids[t] = r;
    strong[t] = gstrong[r];
}

__global__ void band_apply_kernel(int rows, int W, int tiles_x, int tiles_y, const int* __restrict__ perim,
                                  const int* __restrict__ gpar, uint8_t* gstrong,
                                  const uint8_t* __restrict__ strong_edges) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * W || !strong_edges[t]) return;
    bool bottom = t >= W;
    int x = bottom ? t - W : t;
    long long tile = (long long)(bottom ? tiles_y - 1 : 0) * tiles_x + x / HT;
    int node = perim[tile * HP + (bottom ? 64 : 0) + x % HT];
    if (node >= 0) gstrong[gfind_ro(gpar, node)] = 1;
}

// ---------------------------------------------------------------------------
HystLayout hyst_layout(int64_t batch, int H, int W) {
    HystLayout L;
    L.tiles_x = (W + HT - 1) / HT;
    L.tiles_y = (H + HT - 1) / HT;
    L.tiles = batch * (int64_t)L.tiles_x * L.tiles_y;
    L.slots = L.tiles * HP;
    return L;
}

cudaError_t launch_hyst_local(const uint8_t* labels, int64_t batch, int H, int W, uint8_t* final_out,
                              const HystBufs& b, WsHeader* hdr, int sm_count, cudaStream_t st) {
    HystLayout L = hyst_layout(batch, H, W);
    hyst_local_kernel<<<(unsigned)L.tiles, H_THREADS, 0, st>>>(labels, H, W, L.tiles_x, L.tiles_y, final_out,
                                                               b.perim, b.gpar, b.gstrong, b.pending, hdr);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    hyst_merge_kernel<<<(unsigned)L.tiles, 128, 0, st>>>(H, W, L.tiles_x, L.tiles_y, b.perim, b.gpar);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    long long blocks = (L.slots + 255) / 256;
    if (blocks > (long long)sm_count * 16) blocks = (long long)sm_count * 16;
    hyst_resolve_kernel<<<(unsigned)blocks, 256, 0, st>>>(L.slots, b.perim, b.gpar, b.gstrong);
    return cudaGetLastError();
}

cudaError_t launch_hyst_final(const uint8_t* labels, int64_t batch, int H, int W, uint8_t* final_out,
                              const HystBufs& b, cudaStream_t st) {
    HystLayout L = hyst_layout(batch, H, W);
    hyst_final_kernel<<<(unsigned)L.tiles, H_THREADS, 0, st>>>(labels, H, W, L.tiles_x, L.tiles_y, final_out,
                                                               b.gpar, b.gstrong, b.pending);
    return cudaGetLastError();
}

cudaError_t launch_band_edges(int rows, int W, const HystBufs& b, int64_t* ids, uint8_t* strong,
                              cudaStream_t st) {
    HystLayout L = hyst_layout(1, rows, W);
    band_edges_kernel<<<(2 * W + 255) / 256, 256, 0, st>>>(rows, W, L.tiles_x, L.tiles_y, b.perim, b.gpar,
                                                           b.gstrong, ids, strong);
    return cudaGetLastError();
}

cudaError_t launch_band_apply(int rows, int W, const HystBufs& b, const uint8_t* strong_edges,
                              cudaStream_t st) {
    HystLayout L = hyst_layout(1, rows, W);
    band_apply_kernel<<<(2 * W + 255) / 256, 256, 0, st>>>(rows, W, L.tiles_x, L.tiles_y, b.perim, b.gpar,
                                                           b.gstrong, strong_edges);
    return cudaGetLastError();
}

}  // namespace ef
