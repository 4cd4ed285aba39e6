// ef_hyst.cu -- hysteresis edge tracking (trace_edges, hysteresis.py:63-69).
//
// The reference labels 8-connected components of labels != 0 with
// scipy.ndimage.label and keeps those that contain a strong pixel.  The result
// is a set, so any correct connected-component algorithm is bit-exact.  Here
// only the WEAK pixels are labelled: a weak pixel is final iff its component
// among the weak pixels alone touches (8-adjacency) a strong pixel.  (A path
// from a weak pixel to a strong one runs through weak pixels up to the first
// strong pixel it meets; conversely a weak component next to a strong pixel is
// part of that pixel's component.)  Strong pixels are final as they stand (the
// final map is prefilled with them), and a tile reads its neighbours' strong
// bits at its border, so strong pixels never enter the union-find and never
// become border nodes -- on Canny maps half or more of the foreground is
// strong (C3: 52%, C1: 88%).  Input is the two foreground bit planes (label !=
// 0, label == 2); callers with label bytes pack them first (hyst_pack_kernel).
//
//  H1 hyst_local   per 64x64 tile (one warp, or a 128-thread block for dense
//                  tiles / few-tile launches): union-find over the tile's weak
//                  pixels in shared memory; a component is strong if any of
//                  its pixels is next to a strong pixel of the tile or of a
//                  neighbour tile.  Components that do not touch the tile
//                  border are final right away; border-touching ones become
//                  global nodes, numbered tile*256 + (smallest perimeter slot).
//  H2 hyst_merge   unions nodes across tile seams (right, bottom, and the two
//                  diagonal corners) with an atomicCAS union-find in HBM.
//  H3 hyst_resolve propagates "holds a strong pixel" to every node's root.
//  H4 hyst_final   pending weak pixels read their root's strong flag (or the
//                  pending tiles re-run the same tile CCL after an overflow).
//
// The same machinery runs per row band for the multi-GPU partition
// (trace_edges_parallel, hysteresis.py:90-131): band-edge components stay
// pending until the cross-band merge, and strong pixels on a band's edge rows
// are exported to it as strong singletons (read from the strong plane).
#include <algorithm>

#include "ef_common.cuh"
#include "ef_internal.h"
#include "ef_launch.cuh"

namespace ef {

constexpr int HT = 64;          // tile edge
constexpr int HP = 4 * HT;      // perimeter slots per tile
constexpr int H_THREADS = 128;  // 32 pixels per thread: row = tid/2, columns 32*(tid%2) ..
constexpr int NO_POS = 0xffff;  // fits the 16-bit minpos entries

constexpr int LCAP = 256;           // listed foreground pixels per warp (16 rows x 64)
constexpr unsigned NO_SLOT = 0x1ffu;  // info[] slot field: component touches no perimeter slot

struct TileCCL {
    unsigned long long fgrow[HT];  // weak pixels (the union-find's foreground), one word per row
    unsigned long long strow[HT];  // weak pixels next to a strong pixel (component seeds)
    unsigned long long st0[HT];    // strong pixels
    unsigned short par[HT * HT];   // union-find parent; initialised for foreground pixels only
    // per root: bit 15 clear = component holds a strong pixel, bits 0..8 = its
    // smallest perimeter slot (NO_SLOT if interior); 0xffff initially
    unsigned short info[HT * HT];
    unsigned short list[H_THREADS / 32][LCAP];  // each warp's foreground pixels (lane-balanced loops)
    int wcount[H_THREADS / 32];
    int flags;  // 1: any weak pixel, 2: any strong pixel, 4: a warp list overflowed
    int pending;
};

__device__ __forceinline__ bool info_strong(unsigned v) { return !(v & 0x8000u); }
__device__ __forceinline__ unsigned info_slot(unsigned v) { return v & NO_SLOT; }

// info[] entries are 16-bit fields of 32-bit shared-memory words; the updates
// go through shared-space atomics on the containing word (the word address is
// formed as a shared-window address: an integer-cast generic pointer made the
// compiler emit generic atomics, which are slower on shared memory)
__device__ __forceinline__ uint32_t info_word(const unsigned short* p, int& sh) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    sh = (a & 2u) ? 16 : 0;
    return a & ~3u;
}

__device__ __forceinline__ void info_set_strong(unsigned short* p) {
    int sh;
    const uint32_t w = info_word(p, sh);
    asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(w), "r"(~(0x8000u << sh)) : "memory");
}

// lower the slot field to v (CAS on the containing 32-bit word)
__device__ __forceinline__ void info_min_slot(unsigned short* p, unsigned v) {
    int sh;
    const uint32_t w = info_word(p, sh);
    unsigned int old;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(old) : "r"(w) : "memory");
    while (true) {
        const unsigned cur = (old >> sh) & 0xffffu;
        if ((cur & NO_SLOT) <= v) return;
        const unsigned int nw = (old & ~(0xffffu << sh)) | (((cur & ~NO_SLOT) | v) << sh);
        unsigned int seen;
        asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(seen) : "r"(w), "r"(old), "r"(nw) : "memory");
        if (seen == old) return;
        old = seen;
    }
}

__device__ __forceinline__ int sfind(unsigned short* par, int i) {
    while (true) {
        int p = par[i];
        if (p == i) return i;
        int gp = par[p];
        if (gp != p) par[i] = (unsigned short)gp;  // path halving: only ever points further up
        i = p;
    }
}

__device__ __forceinline__ void sunite(unsigned short* par, int a, int b) {
    while (true) {
        a = sfind(par, a);
        b = sfind(par, b);
        if (a == b) return;
        if (a < b) { int t = a; a = b; b = t; }
        if (atomicCAS(&par[a], (unsigned short)a, (unsigned short)b) == (unsigned short)a) return;
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

// One word of a foreground bit plane; 0 outside the frame (or band) rows and words.
__device__ __forceinline__ unsigned long long plane_word(const unsigned long long* __restrict__ plane,
                                                         const FgBits& B, int f, int Y, int rows, int j) {
    return (Y >= 0 && Y < rows && j >= 0 && j < B.words)
               ? __ldg(plane + (unsigned long long)f * B.frame_words + (unsigned long long)Y * B.words + j)
               : 0ull;
}

// Edge bits of the neighbouring words that row Y's weak pixels at columns 0
// and 63 can touch: bit 63 of word j-1 (rows Y-1..Y+1) at bit 0, bit 0 of word
// j+1 at bit 63.  Loaded only where such a weak pixel exists (rare).
__device__ __forceinline__ unsigned long long side_strong(const FgBits& B, int f, int Y, int rows, int j,
                                                          unsigned long long wk) {
    unsigned long long s = 0;
    if (wk & 1ull) {
        const unsigned long long l = plane_word(B.st, B, f, Y - 1, rows, j - 1) |
                                     plane_word(B.st, B, f, Y, rows, j - 1) |
                                     plane_word(B.st, B, f, Y + 1, rows, j - 1);
        s |= l >> 63;
    }
    if (wk >> 63) {
        const unsigned long long r = plane_word(B.st, B, f, Y - 1, rows, j + 1) |
                                     plane_word(B.st, B, f, Y, rows, j + 1) |
                                     plane_word(B.st, B, f, Y + 1, rows, j + 1);
        s |= r << 63;
    }
    return s;
}

// Weak pixels of row Y, word j, and those of them 8-adjacent to a strong pixel
// (the strong plane's rows Y-1..Y+1 dilated by one column, with the edge bits
// of the neighbouring words: another tile's pixels).  Also the strong word.
__device__ __forceinline__ void weak_row(const FgBits& B, int f, int Y, int rows, int j, unsigned long long& wk,
                                         unsigned long long& seed, unsigned long long& st) {
    st = plane_word(B.st, B, f, Y, rows, j);
    wk = plane_word(B.fg, B, f, Y, rows, j) & ~st;
    seed = 0;
    if (wk) {
        const unsigned long long v =
            st | plane_word(B.st, B, f, Y - 1, rows, j) | plane_word(B.st, B, f, Y + 1, rows, j);
        seed = wk & (v | (v << 1) | (v >> 1) | side_strong(B, f, Y, rows, j, wk));
    }
}

// Load this thread's 32-pixel row segment from the bit planes (weak pixels,
// their strong-adjacent seeds, the strong pixels) and publish the tile's row
// words and flags.  Also initialises union-find state for its weak pixels
// (runs inside the 32-pixel segment pre-linked to their start) and appends
// them to the warp's pixel list.  The caller's barrier makes everything visible.
__device__ __forceinline__ void tile_init(TileCCL& s, unsigned long long wk, unsigned long long seed,
                                          unsigned long long strong, bool publish, uint32_t& fg, uint32_t& st);

__device__ __forceinline__ void tile_load(const FgBits& B, int rows, const TileGeo& g, TileCCL& s, uint32_t& fg,
                                          uint32_t& st) {
    const int row = threadIdx.x >> 1;
    unsigned long long wk = 0, seed = 0, strong = 0;
    if (row < g.vh) weak_row(B, g.f, g.y0 + row, rows, g.txi, wk, seed, strong);
    tile_init(s, wk, seed, strong, true, fg, st);
}

// The second half of tile_load: this thread's 32-pixel segment of the row
// words (published to the tile's rows unless they are there already) -> par /
// info / list initialisation and the tile flags.
__device__ __forceinline__ void tile_init(TileCCL& s, unsigned long long wk, unsigned long long seed,
                                          unsigned long long strong, bool publish, uint32_t& fg, uint32_t& st) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int row = tid >> 1, seg = (tid & 1) * 32;
    fg = (uint32_t)(wk >> seg);
    st = (uint32_t)(seed >> seg);
    if (publish) {
        reinterpret_cast<uint32_t*>(&s.fgrow[row])[tid & 1] = fg;
        reinterpret_cast<uint32_t*>(&s.strow[row])[tid & 1] = st;
        reinterpret_cast<uint32_t*>(&s.st0[row])[tid & 1] = (uint32_t)(strong >> seg);
    }
    // warp-exclusive prefix of the foreground counts -> list positions
    const int cnt = __popc(fg);
    int off = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, off, d);
        if (lane >= d) off += v;
    }
    const int total = __shfl_sync(0xffffffffu, off, 31);
    off -= cnt;
    const bool listed = total <= LCAP;
    uint32_t m = fg;
    while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t below = ~fg & ((1u << k) - 1u);
        const int start = below ? (32 - __clz(below)) : 0;  // start of k's run inside the segment
        const int i = row * HT + seg + k;
        s.par[i] = (unsigned short)(row * HT + seg + start);
        s.info[i] = 0xffffu;
        if (listed) s.list[warp][off++] = (unsigned short)i;
    }
    const unsigned any_weak = __any_sync(0xffffffffu, fg != 0);
    const unsigned any_strong = __any_sync(0xffffffffu, (uint32_t)(strong >> seg) != 0u);
    if (lane == 0) {
        s.wcount[warp] = total;
        const int f = (any_weak ? 1 : 0) | (any_strong ? 2 : 0) | (listed ? 0 : 4);
        if (f) atomicOr(&s.flags, f);
    }
}

// Unions of foreground pixel i = (row, x) with its W neighbour across a segment
// seam (runs inside a segment are pre-linked) and its N / NW / NE neighbours.
__device__ __forceinline__ void unite_up(TileCCL& s, int i) {
    const int row = i >> 6, x = i & (HT - 1);
    if ((x & 31) == 0 && x > 0 && ((s.fgrow[row] >> (x - 1)) & 1ull)) sunite(s.par, i, i - 1);
    if (row > 0) {
        const unsigned long long up = s.fgrow[row - 1];
        if ((up >> x) & 1ull) {
            sunite(s.par, i, i - HT);
        } else {
            if (x > 0 && ((up >> (x - 1)) & 1ull)) sunite(s.par, i, i - HT - 1);
            if (x < HT - 1 && ((up >> (x + 1)) & 1ull)) sunite(s.par, i, i - HT + 1);
        }
    }
}

// Root bookkeeping for foreground pixel i whose root is r.
__device__ __forceinline__ void note_root(TileCCL& s, const TileGeo& g, int i, int r) {
    const int row = i >> 6, x = i & (HT - 1);
    if ((s.strow[row] >> x) & 1ull) info_set_strong(&s.info[r]);
    const int p = perim_slot(row, x, g.vh, g.vw);
    if (p != NO_POS) info_min_slot(&s.info[r], (unsigned)p);
}

// General tile CCL (foreground holds weak pixels).  After return par[] holds
// roots for every foreground pixel and info[root] the component's strong flag
// and smallest perimeter slot.  `listed`: every warp's foreground fitted its
// list, so the union / root loops run over the lists with all lanes busy (a
// thin edge leaves most row segments with 0-2 pixels; per-thread loops would
// idle most lanes); otherwise each thread walks its own 32-pixel segment.
__device__ __forceinline__ void tile_ccl(const TileGeo& g, TileCCL& s, uint32_t fg, uint32_t st, bool listed) {
    const int tid = threadIdx.x;
    const int row = tid >> 1, seg = (tid & 1) * 32;
    constexpr int NW = H_THREADS / 32;
    constexpr int RJ = NW * LCAP / H_THREADS;  // list entries per thread at most
    if (listed) {
        int base[NW + 1];
        base[0] = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) base[w + 1] = base[w] + s.wcount[w];
        const int n = base[NW];
        auto entry = [&](int e) -> int {
            int w = 0;
#pragma unroll
            for (int v = 1; v < NW; ++v) w += e >= base[v];
            return s.list[w][e - base[w]];
        };
        for (int e = tid; e < n; e += H_THREADS) unite_up(s, entry(e));
        __syncthreads();
        unsigned short roots[RJ];
#pragma unroll
        for (int j = 0; j < RJ; ++j) {
            const int e = tid + j * H_THREADS;
            if (e < n) {
                const int i = entry(e);
                const int r = sfind(s.par, i);
                roots[j] = (unsigned short)r;
                note_root(s, g, i, r);
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < RJ; ++j) {
            const int e = tid + j * H_THREADS;
            if (e < n) s.par[entry(e)] = roots[j];
        }
        __syncthreads();
        return;
    }
    {
        uint32_t m = fg;
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            unite_up(s, row * HT + seg + k);
        }
    }
    __syncthreads();
    // roots go to registers first: concurrent path halving may still rewrite par[]
    int roots[32];
    {
        uint32_t m = fg;
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            const int i = row * HT + seg + k;
            const int r = sfind(s.par, i);
            roots[k] = r;
            note_root(s, g, i, r);
        }
    }
    __syncthreads();
    {
        uint32_t m = fg;
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            s.par[row * HT + seg + k] = (unsigned short)roots[k];
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Tile-local reach (before the union-find).  A weak component of the tile
// either holds a seed -- then every pixel of it is final -- or it does not;
// the latter decide nothing inside the tile, and only those touching the tile
// perimeter can still be joined to a strong pixel through a neighbour tile.
// Both sets come from a bit-parallel fixpoint over the warp's row words (lane
// = rows 2*lane, 2*lane+1; x = x | dilate8(x) & W, tile-local): typically 1-3
// rounds on Canny maps (C3: 95% of the weak pixels are not reached, 12% touch
// the perimeter).  The union-find then runs only over the perimeter-touching
// unreached components plus the reached pixels on the perimeter (strong
// singletons for the seams), so a perimeter component keeps the node id the
// full CCL gives it (the smallest perimeter slot of the same weak component:
// H4's overflow path re-runs the full CCL and must agree).  More than
// EF_H1_REACH_ITERS rounds (long snakes, mazes): the full sets are kept.
#ifndef EF_H1_REACH
#define EF_H1_REACH 1
#endif

#ifndef EF_H1_REACH_ITERS
#define EF_H1_REACH_ITERS 48
#endif

// rows 2*lane, 2*lane+1 of the tile: weak pixels and their seeds (weak pixels
// 8-adjacent to a strong pixel: the strong rows above and below from the
// neighbouring lanes -- the tiles above / below for lanes 0 and 31 -- and the
// neighbouring words' edge bits only where a weak pixel sits at column 0 or 63)
__device__ __forceinline__ void warp_rows(const FgBits& B, const TileGeo& g, int lane, int H, unsigned long long& f0,
                                          unsigned long long& f1, unsigned long long& s0, unsigned long long& s1) {
    const int ya = g.y0 + 2 * lane;
    // the tile's word column exists (txi < words) and ya >= 0: one 64-bit word index for
    // the lane's four loads, row checks only against the frame's last row
    const unsigned long long w0 =
        (unsigned long long)g.f * B.frame_words + (unsigned long long)ya * (unsigned)B.words + (unsigned)g.txi;
    const bool in0 = ya < H, in1 = ya + 1 < H;
    const unsigned long long t0 = in0 ? __ldg(B.st + w0) : 0ull;
    const unsigned long long t1 = in1 ? __ldg(B.st + w0 + B.words) : 0ull;
    f0 = (in0 ? __ldg(B.fg + w0) : 0ull) & ~t0;
    f1 = (in1 ? __ldg(B.fg + w0 + B.words) : 0ull) & ~t1;
    unsigned long long up = __shfl_up_sync(0xffffffffu, t1, 1), dn = __shfl_down_sync(0xffffffffu, t0, 1);
    if (lane == 0) up = g.y0 > 0 ? __ldg(B.st + w0 - B.words) : 0ull;
    if (lane == 31) dn = g.y0 + HT < H ? __ldg(B.st + w0 + 2 * (unsigned long long)B.words) : 0ull;
    const unsigned long long v0 = up | t0 | t1, v1 = t0 | t1 | dn;
    s0 = f0 ? f0 & (v0 | (v0 << 1) | (v0 >> 1) | side_strong(B, g.f, ya, H, g.txi, f0)) : 0ull;
    s1 = f1 ? f1 & (v1 | (v1 << 1) | (v1 >> 1) | side_strong(B, g.f, ya + 1, H, g.txi, f1)) : 0ull;
}

// x grows inside w by 8-adjacency (tile-local) until it stops changing;
// false if it still changed after EF_H1_REACH_ITERS rounds
__device__ __forceinline__ bool warp_grow(unsigned long long w0, unsigned long long w1, unsigned long long& x0,
                                          unsigned long long& x1, int lane) {
    for (int it = 0; it < EF_H1_REACH_ITERS; ++it) {
        const unsigned long long d0 = x0 | (x0 << 1) | (x0 >> 1), d1 = x1 | (x1 << 1) | (x1 >> 1);
        unsigned long long up = __shfl_up_sync(0xffffffffu, d1, 1), dn = __shfl_down_sync(0xffffffffu, d0, 1);
        if (lane == 0) up = 0;
        if (lane == 31) dn = 0;
        const unsigned long long n0 = w0 & (up | d0 | d1), n1 = w1 & (d0 | d1 | dn);
        const bool ch = ((n0 ^ x0) | (n1 ^ x1)) != 0ull;
        x0 = n0;
        x1 = n1;
        if (!__any_sync(0xffffffffu, ch)) return true;
    }
    return false;
}

// Writes final = 1 for the weak pixels reached from the tile's seeds and, on
// success, narrows (f, s) to the union-find's input: unreached components
// touching the perimeter (f) plus the reached perimeter pixels (f and s).
// Returns false (f, s untouched) when a fixpoint needed too many rounds.
__device__ __forceinline__ bool warp_reach(const TileGeo& g, int lane, uint8_t* __restrict__ fin, int W,
                                           unsigned long long& f0, unsigned long long& f1, unsigned long long& s0,
                                           unsigned long long& s1) {
    unsigned long long r0 = s0, r1 = s1;
    if (!warp_grow(f0, f1, r0, r1, lane)) return false;
    // perimeter of the valid extent: rows 0 and vh-1 whole, else columns 0 and vw-1
    const unsigned long long vmask = g.vw == HT ? ~0ull : ((1ull << g.vw) - 1ull);
    const unsigned long long side = 1ull | (1ull << (g.vw - 1));
    const int ra = 2 * lane, rb = 2 * lane + 1;
    const unsigned long long pm0 = (ra == 0 || ra == g.vh - 1) ? vmask : side;
    const unsigned long long pm1 = (rb == g.vh - 1) ? vmask : side;
    unsigned long long b0 = f0 & ~r0 & pm0, b1 = f1 & ~r1 & pm1;
    if (!warp_grow(f0 & ~r0, f1 & ~r1, b0, b1, lane)) return false;
    // reached pixels are final (weak pixels that join an edge)
    uint8_t* row0 = fin + (size_t)(g.y0 + ra) * W + g.x0;
    for (unsigned long long m = r0; m; m &= m - 1) row0[__ffsll((long long)m) - 1] = 1;
    for (unsigned long long m = r1; m; m &= m - 1) row0[W + __ffsll((long long)m) - 1] = 1;
    f0 = b0 | (r0 & pm0);
    f1 = b1 | (r1 & pm1);
    s0 = r0 & pm0;
    s1 = r1 & pm1;
    return true;
}

// H1: tile-local hysteresis.  Tiles without weak pixels are final as they
// stand (the final map holds their strong pixels) and export nothing; other
// tiles run the shared-memory union-find over their weak pixels and append the
// pixels of undecided border components to the pending list for H4.
// one border-component node into the node list stripe of its tile
__device__ __forceinline__ void append_node(const HystBufs& b, WsHeader* hdr, long long tile, int node) {
    const int stripe = (int)(tile % PL_STRIPES);
    const unsigned long long at = atomicAdd(&b.node_count[stripe], 1ull);
    if (at < b.node_scap) b.node_list[(unsigned long long)stripe * b.node_scap + at] = node;
    else hdr->node_overflow = 1u;
}

__device__ __forceinline__ void hyst_block_tile(const FgBits& B, int H, int W, uint8_t* __restrict__ final_out,
                                                const HystBufs& b, WsHeader* hdr, long long tile, const TileGeo& g,
                                                TileCCL& s, int reach) {
    const int tid = threadIdx.x;
    const int row = tid >> 1, seg = (tid & 1) * 32;
    if (tid == 0) { s.pending = 0; s.flags = 0; }
    uint32_t fg, st;  // this thread's weak pixels and their strong-adjacent seeds
#if EF_H1_REACH
    // warp 0 loads the tile's rows, runs the tile-local reach (final pixels
    // written, the union-find input narrowed) and publishes the rows
    if (tid < 32) {
        unsigned long long f0, f1, s0, s1;
        warp_rows(B, g, tid, H, f0, f1, s0, s1);
        if (reach && __any_sync(0xffffffffu, (f0 | f1) != 0ull))
            warp_reach(g, tid, final_out + (size_t)g.f * H * W, W, f0, f1, s0, s1);
        s.fgrow[2 * tid] = f0;
        s.fgrow[2 * tid + 1] = f1;
        s.strow[2 * tid] = s0;
        s.strow[2 * tid + 1] = s1;
    }
    __syncthreads();
    tile_init(s, s.fgrow[tid >> 1], s.strow[tid >> 1], 0ull, false, fg, st);
#else
    __syncthreads();
    tile_load(B, H, g, s, fg, st);
#endif
    __syncthreads();
    const int flags = s.flags;
    const bool general = flags & 1;  // any weak pixel (else the tile is final as it stands)
    if (general) {
        tile_ccl(g, s, fg, st, !(flags & 4));
        uint32_t fin = 0, pend = 0;
        uint32_t m = fg;
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            const unsigned v = s.info[s.par[row * HT + seg + k]];
            if (info_strong(v)) fin |= 1u << k;
            else if (info_slot(v) != NO_SLOT) pend |= 1u << k;
        }
        if (pend) {
            s.pending = 1;
            const int cnt = __popc(pend);
            const int stripe = (int)(tile % PL_STRIPES);
            unsigned long long at = atomicAdd(&b.plist_count[stripe], (unsigned long long)cnt);
            if (at + cnt > b.plist_scap) {
                hdr->plist_overflow = 1u;
            } else {
                at += (unsigned long long)stripe * b.plist_scap;
                const unsigned long long base =
                    (unsigned long long)g.f * H * W + (unsigned long long)(g.y0 + row) * W + g.x0 + seg;
                int j = 0;
                while (pend) {
                    const int k = __ffs(pend) - 1;
                    pend &= pend - 1;
                    const int root = s.par[row * HT + seg + k];
                    b.plist_idx[at + j] = base + k;
                    b.plist_node[at + j] = (int)(tile * HP) + (int)info_slot(s.info[root]);
                    ++j;
                }
            }
        }
        // weak pixels that join an edge (the final map holds the strong pixels)
        uint8_t* dst = final_out + (size_t)g.f * H * W + (size_t)(g.y0 + row) * W + g.x0 + seg;
        while (fin) {
            const int k = __ffs(fin) - 1;
            fin &= fin - 1;
            EF_DCHECK(row < g.vh && seg + k < g.vw);
            dst[k] = 1;
        }
    }
    // perimeter slots p = tid and tid + 128: node id of the weak component at the slot
    int any_node = 0;
    if (general) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int p = tid + h * H_THREADS;
            int y, x;
            slot_pixel(p, g.vh, g.vw, y, x);
            int node = -1;
            const bool valid = (p < 128) ? (x < g.vw) : (y < g.vh);
            if (valid && y >= 0 && x >= 0 && ((s.fgrow[y] >> x) & 1ull)) {
                const unsigned v = s.info[s.par[y * HT + x]];
                node = (int)(tile * HP) + (int)info_slot(v);
                if (info_slot(v) == (unsigned)p) {
                    b.gpar[node] = node;
                    b.gstrong[node] = info_strong(v) ? 1 : 0;
                    append_node(b, hdr, tile, node);
                }
            }
            b.perim[tile * HP + p] = node;
            any_node |= node >= 0;
        }
    }
    any_node = __syncthreads_or(any_node);
    if (tid == 0) {
        b.border[tile] = any_node ? 1 : 0;
        b.pending[tile] = (uint8_t)s.pending;
        if (s.pending) atomicAdd(&b.pend_tiles[tile % PL_STRIPES], 1ull);
    }
    __syncthreads();  // shared state is reused by the block's next tile
}

__device__ __forceinline__ TileGeo tile_geo_linear(long long tile, int tiles_x, int tiles_y, int H, int W) {
    const int txi = (int)(tile % tiles_x);
    const long long rest = tile / tiles_x;
    return tile_geo_xyz(txi, (int)(rest % tiles_y), (int)(rest / tiles_y), H, W);
}

// H1 for the tiles the warp kernel handed over (more foreground than its
// compact lists hold): one 128-thread block per tile.
__global__ void __launch_bounds__(H_THREADS)
hyst_dense_kernel(FgBits B, int H, int W, int tiles_x, int tiles_y, uint8_t* __restrict__ final_out, HystBufs b,
                  WsHeader* hdr, int reach) {
    __shared__ TileCCL s;
    pdl_wait();
    pdl_trigger();
    const unsigned n = hdr->dense_count;
    for (unsigned e = blockIdx.x; e < n; e += gridDim.x) {
        const long long tile = b.dense[e];
        hyst_block_tile(B, H, W, final_out, b, hdr, tile, tile_geo_linear(tile, tiles_x, tiles_y, H, W), s, reach);
    }
}

// ---------------------------------------------------------------------------
// H1 (warp per tile).  Canny foreground is sparse (C1: ~1% of pixels, ~40 per
// 64x64 tile, a third of the tiles empty), so a tile is one warp's work: row
// bitmasks in shared memory, union-find over COMPACT foreground indices
// (rank of the pixel among the tile's foreground in row-major order, from a
// row prefix count and a popcount), no block barriers.  ~5 KB of shared
// memory per tile instead of ~20 KB.  Tiles with more than WCAP foreground
// pixels go to hyst_dense_kernel.
// ---------------------------------------------------------------------------
#ifndef EF_H1_WCAP
#define EF_H1_WCAP 512
#endif
constexpr int WCAP = EF_H1_WCAP;
#ifndef EF_H1_WARPS
#define EF_H1_WARPS 8
#endif
constexpr int WT_WARPS = EF_H1_WARPS;  // tiles per block (8 measured best with the reach prefilter: 4 -1.7%, 1-2 -2..-4%)

struct WarpTile {
    unsigned long long fgrow[HT];  // weak pixels
    unsigned long long strow[HT];  // weak pixels next to a strong pixel (seeds)
    unsigned short rowbase[HT + 1];
    unsigned short par[WCAP];
    unsigned short info[WCAP];  // as TileCCL::info, per compact index
    unsigned short list[WCAP];  // compact index -> tile pixel (row * 64 + x)
};

__device__ __forceinline__ int cidx(const WarpTile& s, int r, int x) {
    return s.rowbase[r] + __popcll(s.fgrow[r] & ((1ull << x) - 1ull));
}

__device__ __forceinline__ int wfind(const unsigned short* par, int i) {  // read-only
    while (true) {
        const int p = par[i];
        if (p == i) return i;
        i = p;
    }
}

// k-th (0-based) set bit of m
__device__ __forceinline__ int select64(unsigned long long m, int k) {
    int pos = 0;
    uint32_t v = (uint32_t)m;
    int c = __popc(v);
    if (k >= c) {
        k -= c;
        v = (uint32_t)(m >> 32);
        pos = 32;
    }
    c = __popc(v & 0xffffu);
    if (k >= c) { k -= c; v >>= 16; pos += 16; }
    c = __popc(v & 0xffu);
    if (k >= c) { k -= c; v >>= 8; pos += 8; }
    c = __popc(v & 0xfu);
    if (k >= c) { k -= c; v >>= 4; pos += 4; }
    c = __popc(v & 0x3u);
    if (k >= c) { k -= c; v >>= 2; pos += 2; }
    return pos + (k >= (int)(v & 1u) ? 1 : 0);
}

// row holding compact index e (the largest row whose prefix count is <= e)
__device__ __forceinline__ int row_of(const WarpTile& s, int e) {
    int r = 0;
#pragma unroll
    for (int step = 32; step >= 1; step >>= 1)
        if (s.rowbase[r + step] <= e) r += step;
    return r;
}

// BITS: the fused pipeline -- the classifier ORed the foreground / strong
// pixels into bit planes and wrote final = strong, so a tile reads 2 bits per
// pixel instead of its label bytes and stores only weak pixels that join an
// edge.  Otherwise the label bytes are read and the whole final tile written.
// Grid: (ceil(tiles per frame / WT_WARPS), frames); one warp per tile.
__global__ void __launch_bounds__(32 * WT_WARPS)
hyst_local_warp_kernel(FgBits B, int H, int W, int tiles_x, int tiles_y, uint8_t* __restrict__ final_out, HystBufs b,
                       WsHeader* hdr, int reach) {
    extern __shared__ __align__(16) unsigned char h1_smem[];
    WarpTile* tiles = reinterpret_cast<WarpTile*>(h1_smem);  // one per warp (dynamic: up to 16 warps)
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tpf = tiles_x * tiles_y;
    const int t = blockIdx.x * WT_WARPS + warp;
    if (t >= tpf) return;  // warp-uniform; no block barriers below
    WarpTile& s = tiles[warp];
    const int ty = t / tiles_x;
    const TileGeo g = tile_geo_xyz(t - ty * tiles_x, ty, blockIdx.y, H, W);
    const long long tile = (long long)blockIdx.y * tpf + t;
    const int stripe = t % PL_STRIPES;  // == tile % PL_STRIPES only up to the frame offset: any stripe works
    const size_t frame_off = (size_t)g.f * H * W;
    // rows 2*lane, 2*lane+1: weak pixels (f) and their seeds (s)
    unsigned long long f0, f1, s0, s1;
    warp_rows(B, g, lane, H, f0, f1, s0, s1);
    if (!__any_sync(0xffffffffu, (f0 | f1) != 0ull)) {  // final as it stands (the final map holds its strong pixels)
        if (lane == 0) {
            b.border[tile] = 0;
            b.pending[tile] = 0;
        }
        return;
    }
#if EF_H1_REACH
    // tile-local reach: weak pixels joined to a seed inside the tile are final
    // now; of the rest only the components touching the perimeter go on
    if (reach && warp_reach(g, lane, final_out + frame_off, W, f0, f1, s0, s1) &&
        !__any_sync(0xffffffffu, (f0 | f1) != 0ull)) {
        if (lane == 0) {
            b.border[tile] = 0;
            b.pending[tile] = 0;
        }
        return;
    }
#endif
    s.fgrow[2 * lane] = f0;
    s.fgrow[2 * lane + 1] = f1;
    s.strow[2 * lane] = s0;
    s.strow[2 * lane + 1] = s1;
    __syncwarp();
    const int c0 = __popcll(f0), c1 = __popcll(f1);
    int incl = c0 + c1;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
    }
    const int n = __shfl_sync(0xffffffffu, incl, 31);
    if (n > WCAP) {  // dense tile: the block kernel takes it
        if (lane == 0) b.dense[atomicAdd(&hdr->dense_count, 1u)] = (int)tile;
        return;
    }
    bool tile_pending = false;
    {
        const int base0 = incl - c0 - c1;
        s.rowbase[2 * lane] = (unsigned short)base0;
        s.rowbase[2 * lane + 1] = (unsigned short)(base0 + c0);
        if (lane == 31) s.rowbase[HT] = (unsigned short)n;
        __syncwarp();
    }
    {
        // compact list + union-find init, lane-balanced: index e -> (row, column)
        // by the prefix counts; runs are pre-linked to their start
        for (int e = lane; e < n; e += 32) {
            const int r = row_of(s, e);
            const unsigned long long fr = s.fgrow[r];
            const int x = select64(fr, e - s.rowbase[r]);
            const unsigned long long below = ~fr & ((1ull << x) - 1ull);
            const int start = below ? 64 - __clzll((long long)below) : 0;
            EF_DCHECK(e < WCAP && r >= 0 && r < HT && x >= 0 && x < HT && ((fr >> x) & 1ull) && start <= x);
            s.list[e] = (unsigned short)(r * HT + x);
            s.par[e] = (unsigned short)(e - (x - start));
            s.info[e] = 0xffffu;
        }
        __syncwarp();
        // unions with the row above, once per (run, run above) pair: a run's
        // first pixel unites with the runs above touching x-1 .. x+1, every
        // later pixel only with a run above that starts at x+1 (its left
        // neighbour, same component, has covered x-2 .. x)
        for (int e = lane; e < n; e += 32) {
            const int pix = s.list[e];
            const int r = pix >> 6, x = pix & (HT - 1);
            if (r == 0) continue;
            const unsigned long long up = s.fgrow[r - 1];
            const bool in_run = x > 0 && ((s.fgrow[r] >> (x - 1)) & 1ull);
            const bool nx = (up >> x) & 1ull;
            const bool nr = x < HT - 1 && ((up >> (x + 1)) & 1ull);
            EF_DCHECK(!nx || cidx(s, r - 1, x) < n);
            EF_DCHECK(!nr || cidx(s, r - 1, x + 1) < n);
            if (in_run) {
                if (nr && !nx) sunite(s.par, e, cidx(s, r - 1, x + 1));
            } else if (nx) {
                sunite(s.par, e, cidx(s, r - 1, x));
            } else {
                if (x > 0 && ((up >> (x - 1)) & 1ull)) sunite(s.par, e, cidx(s, r - 1, x - 1));
                if (nr) sunite(s.par, e, cidx(s, r - 1, x + 1));
            }
        }
        __syncwarp();
        // roots (read-only finds, so par[e] = root can be written at once) and
        // per-component strong flag (a seed: next to a strong pixel) / smallest perimeter slot
        for (int e = lane; e < n; e += 32) {
            const int pix = s.list[e];
            const int r = pix >> 6, x = pix & (HT - 1);
            const int root = wfind(s.par, e);
            s.par[e] = (unsigned short)root;
            if ((s.strow[r] >> x) & 1ull) info_set_strong(&s.info[root]);
            const int p = perim_slot(r, x, g.vh, g.vw);
            if (p != NO_POS) info_min_slot(&s.info[root], (unsigned)p);
        }
        __syncwarp();
        // final pixels (weak pixels of strong components); undecided border
        // components -> pending list
        for (int e0 = 0; e0 < n; e0 += 32) {
            const int e = e0 + lane;
            bool pend = false;
            int pix = 0;
            unsigned v = 0;
            if (e < n) {
                pix = s.list[e];
                v = s.info[s.par[e]];
                if (info_strong(v)) {
                    EF_DCHECK((pix >> 6) < g.vh && (pix & (HT - 1)) < g.vw);
                    final_out[frame_off + (size_t)(g.y0 + (pix >> 6)) * W + g.x0 + (pix & (HT - 1))] = 1;
                } else {
                    pend = info_slot(v) != NO_SLOT;
                }
            }
            const unsigned pb = __ballot_sync(0xffffffffu, pend);
            if (pb) {
                tile_pending = true;
                unsigned long long at = 0;
                if (lane == 0) at = atomicAdd(&b.plist_count[stripe], (unsigned long long)__popc(pb));
                at = __shfl_sync(0xffffffffu, at, 0);
                if (at + __popc(pb) > b.plist_scap) {
                    if (lane == 0) hdr->plist_overflow = 1u;
                } else if (pend) {
                    const unsigned long long o =
                        (unsigned long long)stripe * b.plist_scap + at + __popc(pb & ((1u << lane) - 1u));
                    b.plist_idx[o] = frame_off + (unsigned long long)(g.y0 + (pix >> 6)) * W + g.x0 + (pix & (HT - 1));
                    b.plist_node[o] = (int)(tile * HP) + (int)info_slot(v);
                }
            }
        }
        __syncwarp();
    }
    // ---- perimeter slots (lane handles slots lane + 32 j): node id of the weak
    // component at each slot; a component's own (smallest) slot makes it a node.
    // A tile without weak pixels on its perimeter writes nothing here: its
    // border flag tells every reader of perim[] (H2, H3's fallback scan, the
    // band-edge export) to skip it.
    const unsigned long long vmask = g.vw == HT ? ~0ull : ((1ull << g.vw) - 1ull);
    const bool per_fg = __any_sync(0xffffffffu, ((f0 | f1) & (1ull | (1ull << (g.vw - 1)))) != 0ull) ||
                        ((s.fgrow[0] | s.fgrow[g.vh - 1]) & vmask) != 0ull;
    if (!per_fg) {
        if (lane == 0) {
            b.border[tile] = 0;
            b.pending[tile] = (uint8_t)tile_pending;
            if (tile_pending) atomicAdd(&b.pend_tiles[stripe], 1ull);
        }
        return;
    }
    int nodes[HP / 32];
    unsigned own[HP / 32];
    int total = 0;
    // the 8 slots' foreground bits from registers: the top / bottom row words
    // (broadcast loads) and this lane's rows lane, lane + 32 (their column 0 /
    // vw-1 bits); only foreground slots look their component up
    unsigned pfg = 0;
    {
        const unsigned long long top = s.fgrow[0] & vmask, bot = s.fgrow[g.vh - 1] & vmask;
        const unsigned long long ra = s.fgrow[lane], rb = s.fgrow[lane + 32];
        pfg |= (unsigned)((top >> lane) & 1ull) | (unsigned)((top >> (lane + 32)) & 1ull) << 1;
        pfg |= (unsigned)((bot >> lane) & 1ull) << 2 | (unsigned)((bot >> (lane + 32)) & 1ull) << 3;
        pfg |= (unsigned)(ra & 1ull) << 4 | (unsigned)(rb & 1ull) << 5;  // rows >= vh hold no foreground
        pfg |= (unsigned)((ra >> (g.vw - 1)) & 1ull) << 6 | (unsigned)((rb >> (g.vw - 1)) & 1ull) << 7;
    }
#pragma unroll
    for (int j = 0; j < HP / 32; ++j) {
        const int p = lane + 32 * j;
        int node = -1;
        bool mine = false;
        if ((pfg >> j) & 1u) {  // a foreground pixel at the slot (the valid extent is in the masks)
            int y, x;
            slot_pixel(p, g.vh, g.vw, y, x);
            const unsigned v = s.info[s.par[cidx(s, y, x)]];
            node = (int)(tile * HP) + (int)info_slot(v);
            if (info_slot(v) == (unsigned)p) {
                mine = true;
                b.gpar[node] = node;
                b.gstrong[node] = info_strong(v) ? 1 : 0;
            }
        }
        EF_DCHECK(p >= 0 && p < HP && (node < 0 || (node >= tile * HP && node < (tile + 1) * HP)));
        b.perim[tile * HP + p] = node;
        nodes[j] = node;
        own[j] = __ballot_sync(0xffffffffu, mine);
        total += __popc(own[j]);
    }
    if (total) {  // one append per tile into its node-list stripe
        unsigned long long at = 0;
        if (lane == 0) at = atomicAdd(&b.node_count[stripe], (unsigned long long)total);
        at = __shfl_sync(0xffffffffu, at, 0);
        if (at + total > b.node_scap) {
            if (lane == 0) hdr->node_overflow = 1u;
        } else {
            unsigned long long o = (unsigned long long)stripe * b.node_scap + at;
#pragma unroll
            for (int j = 0; j < HP / 32; ++j) {
                if ((own[j] >> lane) & 1u) b.node_list[o + __popc(own[j] & ((1u << lane) - 1u))] = nodes[j];
                o += __popc(own[j]);
            }
        }
    }
    if (lane == 0) {
        b.border[tile] = 1;
        b.pending[tile] = (uint8_t)tile_pending;
        if (tile_pending) atomicAdd(&b.pend_tiles[stripe], 1ull);
    }
}

// H2 helpers.  A seam is a pair of 64-vectors held two per lane (v0: index
// lane, v1: index lane + 32); neighbours at index +-1 come by shuffles.
__device__ __forceinline__ void vec_neighbours(int v0, int v1, int lane, int& m0, int& p0, int& m1, int& p1) {
    const int u0 = __shfl_up_sync(0xffffffffu, v0, 1), u1 = __shfl_up_sync(0xffffffffu, v1, 1);
    const int d0 = __shfl_down_sync(0xffffffffu, v0, 1), d1 = __shfl_down_sync(0xffffffffu, v1, 1);
    const int w1 = __shfl_sync(0xffffffffu, v1, 0), w0 = __shfl_sync(0xffffffffu, v0, 31);
    m0 = lane == 0 ? -1 : u0;
    m1 = lane == 0 ? w0 : u1;
    p0 = lane == 31 ? w1 : d0;
    p1 = lane == 31 ? -1 : d1;
}

// unions of A[i] with C[i-1], C[i], C[i+1] (entries < 0: no component).  A
// run of equal A's along the seam unites each C once: the index before has
// already united C[i-1] and C[i].
__device__ __forceinline__ void seam_unite(int* gpar, int a0, int a1, int c0, int c1, int lane) {
    int cm0, cp0, cm1, cp1, am0, ap0, am1, ap1;
    vec_neighbours(c0, c1, lane, cm0, cp0, cm1, cp1);
    vec_neighbours(a0, a1, lane, am0, ap0, am1, ap1);
    auto one = [&](int a, int aprev, int cm, int c, int cp) {
        if (a < 0) return;
        const bool run = a == aprev;
        if (!run && cm >= 0) gunite(gpar, a, cm);
        if (!run && c >= 0 && c != cm) gunite(gpar, a, c);
        if (cp >= 0 && cp != c && cp != cm) gunite(gpar, a, cp);
    };
    one(a0, am0, cm0, c0, cp0);
    one(a1, am1, cm1, c1, cp1);
}

// H2: unions across tile seams, one warp per tile (8 per block; grid
// (ceil(tiles per frame / 8), frames)): the right seam, the bottom seam and
// the two lower corner diagonals.  Tiles without perimeter components -- and
// seams whose other side has none -- are skipped on one byte.  Both seams'
// loads are issued before any union (one round trip, not two), and runs of
// one component along a seam unite once.  Perimeter slots outside the valid
// extent hold -1.
#ifndef EF_H2_WARPS
#define EF_H2_WARPS 8
#endif
constexpr int H2_WARPS = EF_H2_WARPS;  // tiles (warps) per merge block

__global__ void __launch_bounds__(32 * H2_WARPS)
hyst_merge_kernel(int H, int W, int tiles_x, int tiles_y, HystBufs b) {
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tpf = tiles_x * tiles_y;
    const int t = blockIdx.x * 8 + warp;
    if (t >= tpf) return;
    const long long tile = (long long)blockIdx.y * tpf + t;
    const int ty = t / tiles_x, tx = t - ty * tiles_x;
    const bool right = tx + 1 < tiles_x, down = ty + 1 < tiles_y;
    // every load is issued before any is needed (the perimeters of tiles
    // without border components are stale and ignored)
    const int* pa = b.perim + tile * HP;
    const int* pb = b.perim + (right ? tile + 1 : tile) * HP;
    const int* pc = b.perim + (down ? tile + tiles_x : tile) * HP;
    const uint8_t bo = b.border[tile];
    const uint8_t br = right ? b.border[tile + 1] : 0;
    const uint8_t bd = down ? b.border[tile + tiles_x] : 0;
    const int ar0 = pa[192 + lane], ar1 = pa[192 + 32 + lane];  // my right column
    const int cr0 = pb[128 + lane], cr1 = pb[128 + 32 + lane];  // its left column
    const int ad0 = pa[64 + lane], ad1 = pa[64 + 32 + lane];    // my bottom row
    const int cd0 = pc[lane], cd1 = pc[32 + lane];              // its top row
    if (!bo) return;
    int* gpar = b.gpar;
    int ca = -1, cb = -1;  // corner pairs: lane 0 bottom-right, lane 1 bottom-left
    if (lane == 0 && right && down && b.border[tile + tiles_x + 1]) {
        ca = pa[64 + HT - 1];
        cb = b.perim[(tile + tiles_x + 1) * HP + 0];
    }
    if (lane == 1 && tx > 0 && down && b.border[tile + tiles_x - 1]) {
        ca = pa[64 + 0];
        cb = b.perim[(tile + tiles_x - 1) * HP + HT - 1];
    }
    if (br) seam_unite(gpar, ar0, ar1, cr0, cr1, lane);
    if (bd) seam_unite(gpar, ad0, ad1, cd0, cd1, lane);
    if (ca >= 0 && cb >= 0) gunite(gpar, ca, cb);
}

// H3: strong flag of every node onto its root, over the node-list stripes
// (every perimeter slot holding its own id if a stripe overflowed).  Block 0
// also folds the per-stripe counts into the statistics.
__global__ void hyst_resolve_kernel(long long nslots, HystBufs b, WsHeader* hdr) {
    pdl_wait();
    pdl_trigger();
    // grid (x, PL_STRIPES): blockIdx.y is the stripe; on overflow every block
    // row scans a 1/PL_STRIPES share of the perimeter slots instead
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long first = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (hdr->node_overflow) {
        const long long share = (nslots + PL_STRIPES - 1) / PL_STRIPES;
        const long long lo = share * blockIdx.y, hi = min(nslots, lo + share);
        for (long long e = lo + first; e < hi; e += stride) {
            if (!b.border[e / HP]) continue;  // perim[] of a tile without border components is stale
            const int node = b.perim[e];
            if (node != (int)e) continue;  // the node's own (smallest) slot only
            const int r = gfind(b.gpar, node);
            if (b.gstrong[node] && r != node) b.gstrong[r] = 1;
        }
    } else {
        const long long n = (long long)min(b.node_count[blockIdx.y], b.node_scap);
        const int* list = b.node_list + (long long)blockIdx.y * b.node_scap;
        for (long long e = first; e < n; e += stride) {
            const int node = list[e];
            const int r = gfind(b.gpar, node);
            if (b.gstrong[node] && r != node) b.gstrong[r] = 1;
        }
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x < 32) {
        unsigned long long nodes = 0, pend = 0;
        for (int i = threadIdx.x; i < PL_STRIPES; i += 32) {
            nodes += b.node_count[i];
            pend += b.pend_tiles[i];
        }
        for (int d = 16; d; d >>= 1) {
            nodes += __shfl_down_sync(0xffffffffu, nodes, d);
            pend += __shfl_down_sync(0xffffffffu, pend, d);
        }
        if (threadIdx.x == 0) {
            hdr->stats.border_nodes += nodes;
            hdr->stats.pending_tiles += pend;
        }
    }
}

struct TileCCL;
__device__ void hyst_final_tile(const FgBits& B, int H, int W, int tiles_x, int tiles_y,
                                uint8_t* __restrict__ final_out, const HystBufs& b, long long tile, TileCCL& s);

// H4: pixels of undecided border components read their root's strong flag,
// from the pending list.  When the list overflowed (chunks past the cap were
// dropped) the same launch re-runs the tile CCL for every pending tile instead
// (same deterministic CCL, so the same nodes): one kernel either way, no
// always-launched fallback kernel in the PDL chain.
// Grid (x, PL_STRIPES), H_THREADS threads: list mode reads stripe blockIdx.y;
// overflow mode walks the tiles over the flattened grid.
__global__ void __launch_bounds__(H_THREADS)
hyst_final_kernel(FgBits B, int H, int W, int tiles_x, int tiles_y, int frames, uint8_t* __restrict__ final_out,
                  HystBufs b, const WsHeader* __restrict__ hdr) {
    __shared__ TileCCL s;
    pdl_wait();
    pdl_trigger();
    if (!hdr->plist_overflow) {
        const unsigned long long n = min(b.plist_count[blockIdx.y], b.plist_scap);
        const unsigned long long base = (unsigned long long)blockIdx.y * b.plist_scap;
        for (unsigned long long k = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
             k += (unsigned long long)gridDim.x * blockDim.x)
            if (b.gstrong[gfind_ro(b.gpar, b.plist_node[base + k])]) final_out[b.plist_idx[base + k]] = 1;
        return;
    }
    const long long ntiles = (long long)tiles_x * tiles_y * frames;
    const long long nblocks = (long long)gridDim.x * gridDim.y;
    for (long long tile = (long long)blockIdx.y * gridDim.x + blockIdx.x; tile < ntiles; tile += nblocks) {
        if (b.pending[tile]) hyst_final_tile(B, H, W, tiles_x, tiles_y, final_out, b, tile, s);
    }
}

__device__ void hyst_final_tile(const FgBits& B, int H, int W, int tiles_x, int tiles_y,
                                uint8_t* __restrict__ final_out, const HystBufs& b, long long tile, TileCCL& s) {
    const int txi = (int)(tile % tiles_x);
    const long long rest = tile / tiles_x;
    const TileGeo g = tile_geo_xyz(txi, (int)(rest % tiles_y), (int)(rest / tiles_y), H, W);
    if (threadIdx.x == 0) s.flags = 0;
    __syncthreads();
    uint32_t fg, st;
    tile_load(B, H, g, s, fg, st);
    __syncthreads();
    tile_ccl(g, s, fg, st, !(s.flags & 4));
    const int tid = threadIdx.x;
    const int row = tid >> 1, seg = (tid & 1) * 32;
    uint8_t* out = final_out + (size_t)g.f * H * W + (size_t)(g.y0 + row) * W + g.x0 + seg;
    uint32_t m = fg;
    while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        const unsigned v = s.info[s.par[row * HT + seg + k]];
        if (info_strong(v) || info_slot(v) == NO_SLOT) continue;
        const int node = (int)(tile * HP) + (int)info_slot(v);
        if (b.gstrong[gfind_ro(b.gpar, node)]) out[k] = 1;
    }
    __syncthreads();  // shared state is reused by the next tile of this block
}

// Band edge export: component root id and strong flag for the top and bottom
// rows of a band (the frame of `rows` rows).
// Strong pixels are not union-find nodes: a strong pixel on an edge row is
// exported as a strong singleton (id 2^39 + entry, unique inside the band), so
// the cross-band merge makes the weak components next to it strong.
__global__ void band_edges_kernel(int rows, int W, int tiles_x, int tiles_y, const int* __restrict__ perim,
                                  const uint8_t* __restrict__ border, const int* __restrict__ gpar,
                                  const uint8_t* __restrict__ gstrong, FgBits B, int64_t* ids, uint8_t* strong) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * W) return;
    bool bottom = t >= W;
    int x = bottom ? t - W : t;
    long long tile = (long long)(bottom ? tiles_y - 1 : 0) * tiles_x + x / HT;
    int slot = (bottom ? 64 : 0) + x % HT;
    int node = border[tile] ? perim[tile * HP + slot] : -1;
    if (node < 0) {
        const int y = bottom ? rows - 1 : 0;
        const bool st = (__ldg(B.st + (unsigned long long)y * B.words + (x >> 6)) >> (x & 63)) & 1ull;
        ids[t] = st ? (int64_t)((1ll << 39) + t) : -1;
        strong[t] = st ? 1 : 0;
        return;
    }
    int r = gfind_ro(gpar, node);
    ids[t] = r;
    strong[t] = gstrong[r];
}

__global__ void band_apply_kernel(int rows, int W, int tiles_x, int tiles_y, const int* __restrict__ perim,
                                  const uint8_t* __restrict__ border, const int* __restrict__ gpar,
                                  uint8_t* gstrong, const uint8_t* __restrict__ strong_edges) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * W || !strong_edges[t]) return;
    bool bottom = t >= W;
    int x = bottom ? t - W : t;
    long long tile = (long long)(bottom ? tiles_y - 1 : 0) * tiles_x + x / HT;
    if (!border[tile]) return;
    int node = perim[tile * HP + (bottom ? 64 : 0) + x % HT];
    if (node >= 0) gstrong[gfind_ro(gpar, node)] = 1;
}

// ---------------------------------------------------------------------------
// blocks per list stripe for H3 / H4: sm_count / 4 for large launches, fewer
// for small ones (one 512x512 frame has 64 tiles; 2368 blocks were ~3 us each)
static unsigned stripe_blocks(int64_t tiles, int sm_count) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(std::max(1, sm_count / 4), tiles / 256));
}

HystLayout hyst_layout(int64_t batch, int H, int W) {
    HystLayout L;
    L.tiles_x = (W + HT - 1) / HT;
    L.tiles_y = (H + HT - 1) / HT;
    L.tiles = batch * (int64_t)L.tiles_x * L.tiles_y;
    L.slots = L.tiles * HP;
    return L;
}

// H1 for every tile with one 128-thread block per tile (label input): for
// launches with few tiles, where one warp per tile leaves the SMs idle while
// each warp walks a large tile's union-find alone.
__global__ void __launch_bounds__(H_THREADS)
hyst_all_block_kernel(FgBits B, int H, int W, int tiles_x, int tiles_y, long long ntiles,
                      uint8_t* __restrict__ final_out, HystBufs b, WsHeader* hdr, int reach) {
    __shared__ TileCCL s;
    pdl_wait();
    pdl_trigger();
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
        hyst_block_tile(B, H, W, final_out, b, hdr, tile, tile_geo_linear(tile, tiles_x, tiles_y, H, W), s, reach);
}

// Label bytes (0/1/2) -> the two foreground bit planes, one thread per 64-bit
// word (the hysteresis input when no classifier filled the planes: standalone
// tracing, the exact float64 path, the generic classifier).
__global__ void hyst_pack_kernel(const uint8_t* __restrict__ labels, long long rows, int W, int words,
                                 unsigned long long* __restrict__ fg, unsigned long long* __restrict__ st) {
    pdl_wait();
    pdl_trigger();
    const long long n = rows * words;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / words;
        const int j = (int)(i - row * words);
        const uint8_t* p = labels + row * W + 64 * j;
        const int cnt = min(64, W - 64 * j);
        unsigned long long f = 0, s2 = 0;
        if (cnt == 64 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(p) + q);
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    uint32_t a, c;
                    pack4(w4[k], a, c);
                    f |= (unsigned long long)a << (16 * q + 4 * k);
                    s2 |= (unsigned long long)c << (16 * q + 4 * k);
                }
            }
        } else {
            for (int k = 0; k < cnt; ++k) {
                const uint32_t v = p[k];
                f |= (unsigned long long)(v != 0u) << k;
                s2 |= (unsigned long long)(v >= 2u) << k;
            }
        }
        fg[i] = f;
        st[i] = s2;
    }
}

// final = strong for every pixel (the classifier writes this itself in the
// fused path; the hysteresis then adds the weak pixels that join an edge)
__global__ void strong_final_kernel(const uint8_t* __restrict__ labels, long long n, uint8_t* __restrict__ fin) {
    pdl_wait();
    pdl_trigger();
    const bool vec = ((reinterpret_cast<uintptr_t>(labels) | reinterpret_cast<uintptr_t>(fin)) & 15) == 0;
    const long long nv = vec ? n / 16 : 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(labels) + i);
        reinterpret_cast<uint4*>(fin)[i] = make_uint4((v.x >> 1) & 0x01010101u, (v.y >> 1) & 0x01010101u,
                                                      (v.z >> 1) & 0x01010101u, (v.w >> 1) & 0x01010101u);
    }
    for (long long i = nv * 16 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        fin[i] = labels[i] >= 2 ? 1 : 0;
}

// tiles per SM at or below which H1 runs one block per tile (ef_set_block_tile_threshold)
// (initial value: EF_H1_BLOCK_TILES_PER_SM for measurement runs, else 8)
static std::atomic<int> g_block_tiles_per_sm{getenv("EF_H1_BLOCK_TILES_PER_SM") ? atoi(getenv("EF_H1_BLOCK_TILES_PER_SM"))
                                                                               : 8};

void set_block_tile_threshold(int tiles_per_sm) { g_block_tiles_per_sm.store(tiles_per_sm); }

// H1's tile-local reach prefilter (ef_set_tile_reach; EF_H1_REACH=0 in the
// environment starts with it off for measurement runs)
static std::atomic<int> g_tile_reach{getenv("EF_H1_REACH") ? atoi(getenv("EF_H1_REACH")) : 1};

void set_tile_reach(int on) { g_tile_reach.store(on ? 1 : 0); }

cudaError_t launch_hyst_local(const FgBits& B, int64_t batch, int H, int W, uint8_t* final_out, const HystBufs& b,
                              WsHeader* hdr, int sm_count, cudaStream_t st) {
    HystLayout L = hyst_layout(batch, H, W);
    // shared memory bound (~5 KB per warp tile, ~21 KB per dense tile): full carveout
    static std::atomic<uint64_t> configured{0};
    cudaError_t e = once_per_device(configured, [] {
        const int c = (int)cudaSharedmemCarveoutMaxShared;
        cudaError_t r = cudaFuncSetAttribute(hyst_local_warp_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, c);
        if (r == cudaSuccess)
            r = cudaFuncSetAttribute(hyst_local_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(sizeof(WarpTile) * WT_WARPS));
        if (r == cudaSuccess) r = cudaFuncSetAttribute(hyst_dense_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, c);
        if (r == cudaSuccess)
            r = cudaFuncSetAttribute(hyst_all_block_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, c);
        return r;
    });
    if (e != cudaSuccess) return e;
    const bool allblock = L.tiles <= (int64_t)g_block_tiles_per_sm.load() * sm_count;
    const dim3 wgrid((unsigned)((L.tiles_x * L.tiles_y + WT_WARPS - 1) / WT_WARPS), (unsigned)batch);
    if (allblock) {
        // few tiles: a block per tile (the dense-tile list stays empty)
        e = launch_pdl(hyst_all_block_kernel, dim3((unsigned)std::min<int64_t>(L.tiles, 16ll * sm_count)),
                       dim3(H_THREADS), 0, st, B, H, W, L.tiles_x, L.tiles_y, (long long)L.tiles, final_out, b, hdr, g_tile_reach.load());
    } else {
        e = launch_pdl(hyst_local_warp_kernel, wgrid, dim3(32 * WT_WARPS), sizeof(WarpTile) * WT_WARPS, st, B, H, W,
                       L.tiles_x, L.tiles_y,
                       final_out, b, hdr, g_tile_reach.load());
    }
    if (e != cudaSuccess) return e;
    if (!allblock) {  // the block kernel took every tile: the dense list is empty
        e = launch_pdl(hyst_dense_kernel, dim3(sm_count * 4), dim3(H_THREADS), 0, st, B, H, W, L.tiles_x, L.tiles_y,
                       final_out, b, hdr, g_tile_reach.load());
        if (e != cudaSuccess) return e;
    }
    const dim3 mgrid((unsigned)((L.tiles_x * L.tiles_y + H2_WARPS - 1) / H2_WARPS), (unsigned)batch);
    e = launch_pdl(hyst_merge_kernel, mgrid, dim3(32 * H2_WARPS), 0, st, H, W, L.tiles_x, L.tiles_y, b);
    if (e != cudaSuccess) return e;
    return launch_pdl(hyst_resolve_kernel, dim3(stripe_blocks(L.tiles, sm_count), PL_STRIPES), dim3(256), 0, st,
                      (long long)L.slots, b, hdr);
}

cudaError_t launch_hyst_final(const FgBits& B, int64_t batch, int H, int W, uint8_t* final_out, const HystBufs& b,
                              const WsHeader* hdr, int sm_count, cudaStream_t st) {
    HystLayout L = hyst_layout(batch, H, W);
    return launch_pdl(hyst_final_kernel, dim3(stripe_blocks(L.tiles, sm_count), PL_STRIPES), dim3(H_THREADS), 0,
                      st, B, H, W, L.tiles_x, L.tiles_y, (int)batch, final_out, b, hdr);
}

cudaError_t launch_hyst_pack(const uint8_t* labels, int64_t batch, int H, int W, const FgBits& B, int sm_count,
                             cudaStream_t st) {
    const long long n = batch * (long long)H * B.words;
    const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 8ll * sm_count));
    return launch_pdl(hyst_pack_kernel, dim3(grid), dim3(256), 0, st, labels, batch * (long long)H, W, B.words, B.fg,
                      B.st);
}

cudaError_t launch_strong_final(const uint8_t* labels, long long n, uint8_t* fin, int sm_count, cudaStream_t st) {
    const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>((n / 16 + 255) / 256, 8ll * sm_count));
    return launch_pdl(strong_final_kernel, dim3(grid), dim3(256), 0, st, labels, n, fin);
}

cudaError_t launch_band_edges(int rows, int W, const HystBufs& b, const FgBits& B, int64_t* ids, uint8_t* strong,
                              cudaStream_t st) {
    HystLayout L = hyst_layout(1, rows, W);
    band_edges_kernel<<<(2 * W + 255) / 256, 256, 0, st>>>(rows, W, L.tiles_x, L.tiles_y, b.perim, b.border, b.gpar,
                                                           b.gstrong, B, ids, strong);
    return cudaGetLastError();
}

cudaError_t launch_band_apply(int rows, int W, const HystBufs& b, const uint8_t* strong_edges,
                              cudaStream_t st) {
    HystLayout L = hyst_layout(1, rows, W);
    band_apply_kernel<<<(2 * W + 255) / 256, 256, 0, st>>>(rows, W, L.tiles_x, L.tiles_y, b.perim, b.border, b.gpar,
                                                           b.gstrong, strong_edges);
    return cudaGetLastError();
}

}  // namespace ef
