// ef_internal.h -- launcher declarations shared by the .cu files.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "ef_common.cuh"  // EF_DCHECK

namespace ef {

struct ExactParams;
struct FastParams;
struct WsHeader;

// geometry of one frame or one row band of a frame (see ef_band_* in the ABI)
struct FrameGeom {
    int H;       // rows held in the source buffer
    int W;       // columns
    int g0;      // global row of source row 0
    int full_H;  // rows of the whole frame (clamping is against [0, full_H))
    int out0;    // first global row to classify
    int rows;    // rows to classify; output row (Y - out0)
    // Peer halos (multi-GPU row bands, ef_band_canny_u8_peer): when set, the
    // source buffer holds only rows [out0, out0 + rows); rows above come from
    // `top` (first row = global row g0) and rows below from `bot` (first row =
    // global row out0 + rows) -- neighbour bands read in place, over NVLink
    // for another GPU's HBM.  nullptr: the source holds rows [g0, g0 + H).
    const uint8_t* top = nullptr;
    const uint8_t* bot = nullptr;
};

#ifdef __CUDACC__
// Kernels reading input rows are compiled twice: PEER = false (one contiguous
// source buffer: no peer checks anywhere in the code) and PEER = true (band
// calls with peer halos).
// first global row held at the source pointer
template <bool PEER>
__host__ __device__ __forceinline__ int src_row0(const FrameGeom& g) { return PEER ? g.out0 : g.g0; }
// rows addressable from the source pointer (the tensor map's extent)
__host__ __device__ __forceinline__ int src_rows(const FrameGeom& g) { return (g.top || g.bot) ? g.rows : g.H; }
// global row y (inside [g0, g0 + H)) of frame `img` (= source + frame offset)
template <bool PEER>
__device__ __forceinline__ const uint8_t* frame_row(const uint8_t* img, const FrameGeom& g, int y) {
    if (PEER) {
        if (g.top && y < g.out0) return g.top + (size_t)(y - g.g0) * g.W;
        if (g.bot && y >= g.out0 + g.rows) return g.bot + (size_t)(y - g.out0 - g.rows) * g.W;
    }
    return img + (size_t)(y - src_row0<PEER>(g)) * g.W;
}
#endif

struct HystLayout {
    int tiles_x, tiles_y;
    int64_t tiles, slots;
};

constexpr int PL_STRIPES = 64;  // pending-list stripes (tile % 64): spreads the append counters

struct HystBufs {
    int* perim;
    int* gpar;
    uint8_t* gstrong;
    uint8_t* pending;
    uint8_t* border;  // per tile: some perimeter slot holds a component (H1 -> H2)
    unsigned long long* plist_idx;  // pixels of undecided border components (H1 -> H4),
    int* plist_node;                //   PL_STRIPES stripes of plist_scap entries
    unsigned long long* plist_count;  // per stripe
    unsigned long long plist_scap;
    int* node_list;                  // border-component nodes (H1 -> H3), PL_STRIPES stripes of node_scap
    unsigned long long* node_count;  // per stripe
    unsigned long long node_scap;
    unsigned long long* pend_tiles;  // per stripe: tiles with undecided border components (statistics)
    int* dense;  // tiles too dense for the warp kernel (one entry per tile at most)
};

// Foreground bit planes for the fused pipeline (ef_canny_u8): the classifier
// ORs every foreground / strong pixel into row-major bit planes (one bit per
// pixel, 64-bit words), so hysteresis reads 2 bits per pixel instead of
// rescanning the label bytes (about 1% of Canny labels are foreground).
// fg == nullptr: planes off.
struct FgBits {
    unsigned long long* fg;
    unsigned long long* st;
    int words;                     // words per output row: ceil(W / 64)
    unsigned long long frame_words;  // words per frame: rows * words
    long long fin_off;             // final map - label map (bytes): the classifier also writes final = strong
};

#ifdef __CUDACC__
// pixels x .. x+3 (x % 4 == 0) of output row yo in frame f: nibbles of fg / strong bits
__device__ __forceinline__ void fg_bits_or(const FgBits& B, unsigned long long f, int yo, int x, uint32_t fgn,
                                           uint32_t stn) {
    const unsigned long long w = f * B.frame_words + (unsigned long long)yo * B.words + (unsigned)(x >> 6);
    EF_DCHECK(B.st - B.fg >= 0 && w < (unsigned long long)(B.st - B.fg) && (x & 3) == 0 && (unsigned)(x >> 6) < (unsigned)B.words);
    // global-space reductions (no return value): stated explicitly -- through
    // pointers the compiler could not prove global (an out-of-line classifier)
    // these compiled to generic atomics with shared-space checks (K1 +3%)
    if (fgn)
        asm volatile("red.global.or.b64 [%0], %1;" ::"l"(B.fg + w), "l"((unsigned long long)fgn << (x & 63)) : "memory");
    if (stn)
        asm volatile("red.global.or.b64 [%0], %1;" ::"l"(B.st + w), "l"((unsigned long long)stn << (x & 63)) : "memory");
}

// 4-byte global store (explicit state space: see fg_bits_or)
__device__ __forceinline__ void st_global_u32(void* p, uint32_t v) {
    asm volatile("st.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
#endif

size_t ex_smem_bytes(int r);
size_t k1_smem_bytes(int r);

template <typename In>
cudaError_t launch_exact(const In* src, int64_t batch, int H, int W, const ExactParams& P,
                         uint8_t* labels, double* blurred, double* gx, double* gy, double* mag,
                         int64_t* ori, double* thin, unsigned long long* max_bits, WsHeader* hdr,
                         cudaStream_t st);

// B.fg != nullptr only where k1_emits_bits() holds
cudaError_t launch_k1(const uint8_t* src, int64_t batch, const FrameGeom& g, const FastParams& P,
                      uint8_t* labels, unsigned long long* fix_list, WsHeader* hdr, const FgBits& B,
                      cudaStream_t st);
bool k1_emits_bits(const FastParams& P, const FrameGeom& g);

cudaError_t launch_k1v1(const uint8_t* src, int64_t batch, const FrameGeom& g, const FastParams& P,
                        uint8_t* labels, unsigned long long* fix_list, WsHeader* hdr, cudaStream_t st);
cudaError_t launch_k1v2(const uint8_t* src, int64_t batch, const FrameGeom& g, const FastParams& P,
                        uint8_t* labels, unsigned long long* fix_list, WsHeader* hdr, const FgBits& B,
                        cudaStream_t st);
bool k1v2_supported(const FastParams& P, const FrameGeom& g);

cudaError_t launch_fix(const uint8_t* src, int64_t batch, const FrameGeom& g, const ExactParams& P,
                       uint8_t* labels, const unsigned long long* list, WsHeader* hdr, const FgBits& B,
                       int sm_count, cudaStream_t st);

HystLayout hyst_layout(int64_t batch, int H, int W);
// Hysteresis over the foreground bit planes B (label != 0, label == 2), with
// final_out already holding final = strong: H1 (+ dense tiles), H2, H3.
cudaError_t launch_hyst_local(const FgBits& B, int64_t batch, int H, int W, uint8_t* final_out, const HystBufs& b,
                              WsHeader* hdr, int sm_count, cudaStream_t st);
// H4: pending weak pixels read their root's flag
cudaError_t launch_hyst_final(const FgBits& B, int64_t batch, int H, int W, uint8_t* final_out, const HystBufs& b,
                              const WsHeader* hdr, int sm_count, cudaStream_t st);
// label bytes -> bit planes; final = strong (callers without the fused classifier)
cudaError_t launch_hyst_pack(const uint8_t* labels, int64_t batch, int H, int W, const FgBits& B, int sm_count,
                             cudaStream_t st);
cudaError_t launch_strong_final(const uint8_t* labels, long long n, uint8_t* fin, int sm_count, cudaStream_t st);
cudaError_t launch_band_edges(int rows, int W, const HystBufs& b, const FgBits& B, int64_t* ids, uint8_t* strong,
                              cudaStream_t st);
cudaError_t launch_band_apply(int rows, int W, const HystBufs& b, const uint8_t* strong_edges,
                              cudaStream_t st);
void set_block_tile_threshold(int tiles_per_sm);
void set_tile_reach(int on);

size_t band_merge_scratch_bytes(int nbands, int W);
cudaError_t launch_band_merge(int nbands, int W, const int64_t* ids, const uint8_t* strong, uint8_t* out,
                              void* scratch, cudaStream_t st);

cudaError_t launch_nms(const double* mag, const int64_t* ori, int H, int W, double* thin, int* bad, cudaStream_t st);
cudaError_t launch_threshold(const double* thin, long long n, double low, double high, uint8_t* labels,
                             cudaStream_t st);
cudaError_t launch_quantize(const double* gx, const double* gy, long long n, int64_t* ori, cudaStream_t st);
cudaError_t launch_laplacian(const double* src, int H, int W, double* out, cudaStream_t st);

}  // namespace ef
