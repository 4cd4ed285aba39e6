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
    unsigned long long fgrow[HT];  // foreground (label != 0) bit per pixel, one word per row
    unsigned long long strow[HT];  // strong bit per pixel
    int par[HT * HT];              // union-find parent; initialised for foreground pixels only
    int minpos[HT * HT];           // smallest perimeter slot per root (foreground only)
    unsigned char sflag[HT * HT];  // component holds a strong pixel (per root)
    int pending;
    int nodes;
    int any;
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

// Tiles are launched on a (tiles_x, tiles_y, frames) grid: no index division.
__device__ __forceinline__ TileGeo tile_geo_xyz(int txi, int tyi, int f, int H, int W) {
    TileGeo g;
    g.f = f;
    g.tyi = tyi;
    g.txi = txi;
    g.y0 = g.tyi * HT;
    g.x0 = g.txi * HT;
    g.vh = min(HT, H - g.y0);
    g.vw = min(HT, W - g.x0);
    return g;
}

__device__ __forceinline__ long long tile_id_xyz(int tiles_x, int tiles_y) {
    return ((long long)blockIdx.z * tiles_y + blockIdx.y) * tiles_x + blockIdx.x;
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

// Pack the foreground / strong bits of 4 label bytes (values 0/1/2) into nibbles.
__device__ __forceinline__ void pack4(uint32_t w, uint32_t& fg, uint32_t& st) {
    const uint32_t nz = (w | (w >> 1)) & 0x01010101u;
    const uint32_t sg = (w >> 1) & 0x01010101u;
    fg = (nz * 0x10204080u) >> 28;
    st = (sg * 0x10204080u) >> 28;
}

// Shared tile CCL used by H1 and H4.  Work is proportional to the foreground:
// label bytes become per-row bit masks, union-find runs over foreground pixels
// only.  After return (and a barrier) par[] holds roots for every foreground
// pixel, sflag[root] marks strong components and minpos[root] the smallest
// perimeter slot (NO_POS if interior).  Returns this thread's 16-bit
// foreground mask (row = tid/4, columns 16*(tid%4) ..).
__device__ uint32_t tile_ccl(const uint8_t* __restrict__ labels, int H, int W, const TileGeo& g, TileCCL& s) {
    const int tid = threadIdx.x;
    const int row = tid >> 2, seg = (tid & 3) * 16;
    const uint8_t* frame = labels + (size_t)g.f * H * W;
    const int Y = g.y0 + row;
    uint32_t words[4] = {0u, 0u, 0u, 0u};
    const uint8_t* src = frame + (size_t)Y * W + g.x0 + seg;
    if (row < g.vh && seg + 16 <= g.vw && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
        uint4 q = __ldg(reinterpret_cast<const uint4*>(src));
        words[0] = q.x; words[1] = q.y; words[2] = q.z; words[3] = q.w;
    } else if (row < g.vh) {
        for (int k = 0; k < 16; ++k)
            if (seg + k < g.vw) words[k >> 2] |= (uint32_t)src[k] << (8 * (k & 3));
    }
    uint32_t fg = 0, st = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        uint32_t f, t;
        pack4(words[j], f, t);
        fg |= f << (4 * j);
        st |= t << (4 * j);
    }
    if (tid == 0) s.any = 0;
    // segment masks -> row words (4 threads per row, 16 bits each)
    reinterpret_cast<unsigned short*>(&s.fgrow[row])[tid & 3] = (unsigned short)fg;
    reinterpret_cast<unsigned short*>(&s.strow[row])[tid & 3] = (unsigned short)st;
    // init only foreground pixels; runs inside the segment pre-linked to their start
    {
        uint32_t m = fg;
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            const int i = row * HT + seg + k;
            const bool left_in_run = k > 0 && ((fg >> (k - 1)) & 1u);
            int start = k;
            if (left_in_run) {  // start of the run containing k inside this segment
                const uint32_t below = ~fg & ((1u << k) - 1u);
                start = below ? (32 - __clz(below)) : 0;
            }
            s.par[i] = row * HT + seg + start;
            s.minpos[i] = NO_POS;
            s.sflag[i] = 0;
        }
    }
    const int any = __syncthreads_or(fg != 0);
    if (!any) return 0;
    // unions: W across segments, N / NW / NE from the row above (bit tests)
    const unsigned long long up = row > 0 ? s.fgrow[row - 1] : 0ull;
    const unsigned long long cur = s.fgrow[row];
    {
        uint32_t m = fg;
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            const int x = seg + k, i = row * HT + x;
            if (k == 0 && x > 0 && ((cur >> (x - 1)) & 1ull)) sunite(s.par, i, i - 1);
            if (up) {
                if ((up >> x) & 1ull) {
                    sunite(s.par, i, i - HT);
                } else {
                    if (x > 0 && ((up >> (x - 1)) & 1ull)) sunite(s.par, i, i - HT - 1);
                    if (x < HT - 1 && ((up >> (x + 1)) & 1ull)) sunite(s.par, i, i - HT + 1);
                }
            }
        }
    }
    __syncthreads();
    // roots into registers first (concurrent path halving may rewrite par[])
    int roots[16];
    {
        uint32_t m = fg;
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            const int x = seg + k, i = row * HT + x;
            const int r = sfind(s.par, i);
            roots[k] = r;
            if ((st >> k) & 1u) s.sflag[r] = 1;
            const int p = perim_slot(row, x, g.vh, g.vw);
            if (p != NO_POS) atomicMin(&s.minpos[r], p);
        }
    }
    __syncthreads();
    {
        uint32_t m = fg;
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            s.par[row * HT + seg + k] = roots[k];
        }
    }
    __syncthreads();
    return fg;
}

// 16 bits -> 16 bytes (0/1)
__device__ __forceinline__ uint4 expand16(uint32_t bits) {
    uint4 o;
    o.x = ((bits & 0xFu) * 0x00204081u) & 0x01010101u;
    o.y = (((bits >> 4) & 0xFu) * 0x00204081u) & 0x01010101u;
    o.z = (((bits >> 8) & 0xFu) * 0x00204081u) & 0x01010101u;
    o.w = (((bits >> 12) & 0xFu) * 0x00204081u) & 0x01010101u;
    return o;
}

__device__ __forceinline__ void store16(uint8_t* dst, int valid, uint4 o) {
    if (valid >= 16 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        *reinterpret_cast<uint4*>(dst) = o;
    } else {
        const uint32_t w[4] = {o.x, o.y, o.z, o.w};
        for (int k = 0; k < valid && k < 16; ++k) dst[k] = (uint8_t)(w[k >> 2] >> (8 * (k & 3)));
    }
}

__global__ void __launch_bounds__(H_THREADS)
hyst_local_kernel(const uint8_t* __restrict__ labels, int H, int W, int tiles_x, int tiles_y,
                  uint8_t* __restrict__ final_out, int* __restrict__ perim, int* __restrict__ gpar,
                  uint8_t* __restrict__ gstrong, uint8_t* __restrict__ pending, WsHeader* hdr) {
    __shared__ TileCCL s;
    const long long tile = tile_id_xyz(tiles_x, tiles_y);
    TileGeo g = tile_geo_xyz(blockIdx.x, blockIdx.y, blockIdx.z, H, W);
    if (threadIdx.x == 0) { s.pending = 0; s.nodes = 0; }
    const uint32_t fg = tile_ccl(labels, H, W, g, s);
    const int tid = threadIdx.x;
    const int row = tid >> 2, seg = (tid & 3) * 16;
    uint32_t fin = 0;
    bool pend = false;
    {
        uint32_t m = fg;
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            const int root = s.par[row * HT + seg + k];
            if (s.sflag[root]) fin |= 1u << k;
            else if (s.minpos[root] != NO_POS) pend = true;
        }
    }
    if (row < g.vh && seg < g.vw)
        store16(final_out + (size_t)g.f * H * W + (size_t)(g.y0 + row) * W + g.x0 + seg, g.vw - seg, expand16(fin));
    if (pend) s.pending = 1;
    // perimeter slot tid: node id of the component at that slot, -1 if background
    {
        const int p = tid;  // H_THREADS == HP
        int y, x;
        slot_pixel(p, g.vh, g.vw, y, x);
        int node = -1;
        const bool valid = (p < 128) ? (x < g.vw) : (y < g.vh);
        if (valid && y >= 0 && x >= 0 && ((s.fgrow[y] >> x) & 1ull)) {
            const int root = s.par[y * HT + x];
            node = (int)(tile * HP) + s.minpos[root];
            if (s.minpos[root] == p) {
                gpar[node] = node;
                gstrong[node] = s.sflag[root];
                atomicAdd(&s.nodes, 1);
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
    const long long tile = tile_id_xyz(tiles_x, tiles_y);
    TileGeo g = tile_geo_xyz(blockIdx.x, blockIdx.y, blockIdx.z, H, W);
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
                TileGeo gc = tile_geo_xyz(blockIdx.x, blockIdx.y + 1, blockIdx.z, H, W);
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
    const long long tile = tile_id_xyz(tiles_x, tiles_y);
    if (!pending[tile]) return;
    TileGeo g = tile_geo_xyz(blockIdx.x, blockIdx.y, blockIdx.z, H, W);
    const uint32_t fg = tile_ccl(labels, H, W, g, s);
    const int tid = threadIdx.x;
    const int row = tid >> 2, seg = (tid & 3) * 16;
    uint32_t m = fg;
    uint8_t* out = final_out + (size_t)g.f * H * W + (size_t)(g.y0 + row) * W + g.x0 + seg;
    while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        const int root = s.par[row * HT + seg + k];
        if (s.sflag[root] || s.minpos[root] == NO_POS) continue;
        const int node = (int)(tile * HP) + s.minpos[root];
        if (gstrong[gfind_ro(gpar, node)]) out[k] = 1;
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
    const dim3 tgrid(L.tiles_x, L.tiles_y, (unsigned)batch);
    hyst_local_kernel<<<tgrid, H_THREADS, 0, st>>>(labels, H, W, L.tiles_x, L.tiles_y, final_out,
                                                               b.perim, b.gpar, b.gstrong, b.pending, hdr);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    hyst_merge_kernel<<<tgrid, 128, 0, st>>>(H, W, L.tiles_x, L.tiles_y, b.perim, b.gpar);
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
    const dim3 tgrid(L.tiles_x, L.tiles_y, (unsigned)batch);
    hyst_final_kernel<<<tgrid, H_THREADS, 0, st>>>(labels, H, W, L.tiles_x, L.tiles_y, final_out,
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
