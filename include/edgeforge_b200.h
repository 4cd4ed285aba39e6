/*
 * edgeforge_b200.h -- C ABI of the B200-native Canny path (libedgeforge_b200.so).
 *
 * The reference (edgeforge, pure Python) has no FFI or plugin registry; its
 * seam is the Python call run_pipeline(img, PipelineConfig) and the stage
 * functions it sequences.  Each entry point below replaces one of those
 * reference interfaces (cited as file:line under /root/reference/pkg/src/edgeforge)
 * and is what a ctypes / cffi / cgo binding of that seam binds.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "d_" pointers are CUDA device pointers
 *    owned by the caller; "h_" pointers are host pointers.
 *  - Images are dense row-major frames: frame f, row y, column x lives at
 *    base + (f*height + y)*width + x.  batch >= 1 frames of height x width.
 *  - weights: HOST pointer to the 2*radius+1 float64 Gaussian weights, exactly
 *    GaussianKernel.weights (filtering.py:14-29): symmetric, summing to 1.
 *  - low/high: absolute thresholds on the raw Sobel magnitude (Thresholds,
 *    hysteresis.py:26-33): 0 <= low <= high.
 *  - labels: u8 {0 none, 1 weak, 2 strong} (hysteresis.py:19-21);
 *    final: u8 {0,1}, the traced edge set (EdgeMap.final as bytes).
 *  - stream: a cudaStream_t passed as void*; all device work is stream-ordered
 *    and asynchronous unless stated otherwise.
 *  - Return value: 0 on success; EF_EINVAL (-1) for invalid arguments (the
 *    reference raises ValueError), EF_ECUDA (-2) for CUDA failures, EF_ENOMEM
 *    (-3) when the workspace is too small.  ef_last_error() describes the last
 *    failure on the calling thread.
 *  - Thread safety: concurrent calls are safe if each thread uses its own
 *    stream and workspace.
 */
#ifndef EDGEFORGE_B200_H
#define EDGEFORGE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EF_ABI_VERSION 1
#define EF_OK 0
#define EF_EINVAL (-1)
#define EF_ECUDA (-2)
#define EF_ENOMEM (-3)
#define EF_MAX_RADIUS 15

/* Library / error plumbing. */
int ef_abi_version(void);
const char* ef_last_error(void);

/* Per-call statistics, accumulated on the device into the workspace and read
 * back (synchronously) by ef_read_stats. */
typedef struct ef_stats {
    int64_t fixups;           /* pixels whose fp32 decision was not certified and
                                 were recomputed in exact float64               */
    int64_t ambiguous;        /* orientation within 1e-12 of a sector boundary:
                                 resolved with the reference's atan2 formula    */
    int64_t border_nodes;     /* tile-border components entering the union-find */
    int64_t pending_tiles;    /* tiles finalised after the global merge         */
} ef_stats;

/* Hysteresis tuning (process-wide): launches with at most tiles_per_sm 64x64
 * tiles per SM run the tile pass with one 128-thread block per tile instead of
 * one warp per tile (few, large tiles: C0).  Default 8; 0 = always one
 * warp per tile.  The result is identical either way. */
int ef_set_block_tile_threshold(int32_t tiles_per_sm);

/* Hysteresis tuning: 1 (default) = the tile pass first grows the weak pixels
 * reached from the tile's seeds (final at once) and runs its union-find only
 * over the unreached components touching the tile perimeter; 0 = union-find
 * over every weak pixel.  The result is identical either way. */
int ef_set_tile_reach(int32_t on);

/* Which capacity fallbacks the last call on this workspace took (synchronises
 * `stream`): h_out[0] fix list overflowed (FX scanned every label), [1] a
 * pending-list stripe overflowed (H4 re-ran the pending tiles), [2] tiles H1's
 * warp kernel handed to the block kernel, [3] a node-list stripe overflowed (H3
 * scanned every perimeter slot).  For tests and diagnostics. */
int ef_read_paths(const void* d_workspace, size_t workspace_bytes, void* stream, uint32_t* h_out);

/* Bytes of device workspace needed by ef_canny_u8 / ef_canny_f64 /
 * ef_trace_edges for `batch` frames of height x width. */
size_t ef_workspace_bytes(int64_t batch, int32_t height, int32_t width);

/* Zero the statistics block of a workspace (stream-ordered). */
int ef_reset_stats(void* d_workspace, size_t workspace_bytes, void* stream);
/* Synchronise `stream` and copy the statistics out. */
int ef_read_stats(const void* d_workspace, size_t workspace_bytes, void* stream, ef_stats* h_out);

/* Instrumentation (no reference counterpart): CUDA events (cudaEvent_t, or
 * NULL to stop) that this thread's later classify launches -- ef_classify_u8,
 * ef_canny_u8, ef_band_canny_u8 -- record on their stream right before the
 * classifier kernel and right after its fix-up kernels. */
int ef_set_classify_events(void* start_event, void* stop_event);

/* Whole Canny path for u8 frames on the device -- replaces run_pipeline
 * (bench.py:61-126, operator="canny", explicit Thresholds) for inputs whose
 * pixels are integers in [0,255] (GrayImage holds them as float64, image.py:23-50).
 *   gaussian_blur (filtering.py:66-91) + sobel (gradient.py:73-90)
 *   + non_max_suppress (nms.py:36-55) + double_threshold (hysteresis.py:54-60)
 *   -> d_labels;  trace_edges (hysteresis.py:63-69) -> d_final.
 * Fused fp32 stencil with a certified error bound; pixels whose decision is
 * inside the bound are recomputed in exact float64 in the reference's
 * operation order, so d_labels/d_final are bit-identical to the reference. */
int ef_canny_u8(const uint8_t* d_src, int64_t batch, int32_t height, int32_t width,
                const double* h_weights, int32_t radius, double low, double high,
                uint8_t* d_labels, uint8_t* d_final, void* d_workspace,
                size_t workspace_bytes, void* stream);

/* Same path for arbitrary finite float64 pixels (GrayImage.pixels) -- exact
 * float64 stencil in reference order on the GPU (no fp32 fast path). */
int ef_canny_f64(const double* d_src, int64_t batch, int32_t height, int32_t width,
                 const double* h_weights, int32_t radius, double low, double high,
                 uint8_t* d_labels, uint8_t* d_final, void* d_workspace,
                 size_t workspace_bytes, void* stream);

/* Stage 1-4 only (labels, no tracing): the fused classify kernel.
 * Replaces gaussian_blur + sobel + non_max_suppress + double_threshold. */
int ef_classify_u8(const uint8_t* d_src, int64_t batch, int32_t height, int32_t width,
                   const double* h_weights, int32_t radius, double low, double high,
                   uint8_t* d_labels, void* d_workspace, size_t workspace_bytes, void* stream);

/* Hysteresis only -- replaces trace_edges (hysteresis.py:63-69): 8-connected
 * components of labels != 0 that contain a strong pixel. */
int ef_trace_edges(const uint8_t* d_labels, int64_t batch, int32_t height, int32_t width,
                   uint8_t* d_final, void* d_workspace, size_t workspace_bytes, void* stream);

/* Every float64 intermediate of one frame (keep_intermediates=True,
 * bench.py:124-125): blurred (GrayImage), gx, gy, magnitude, orientation
 * (int64 degrees, GradientField gradient.py:19-34), thinned (ThinnedField,
 * nms.py:13-24) and labels.  Input is u8 (d_src8) or float64 (d_src64); the
 * other pointer must be NULL.  Any output pointer may be NULL. */
int ef_stages_f64(const uint8_t* d_src8, const double* d_src64, int32_t height, int32_t width,
                  const double* h_weights, int32_t radius, double low, double high,
                  double* d_blurred, double* d_gx, double* d_gy, double* d_magnitude,
                  int64_t* d_orientation, double* d_thinned, uint8_t* d_labels, void* stream);

/* Exact float64 maximum of the thinned field of one frame -- the reduction in
 * auto_thresholds (bench.py:51-58).  Writes one double to d_max. */
int ef_thinned_max(const uint8_t* d_src8, const double* d_src64, int32_t height, int32_t width,
                   const double* h_weights, int32_t radius, double* d_max, void* stream);

/* Stage-level kernels for the reference's stage API on arbitrary arrays. */
/* non_max_suppress (nms.py:36-55) on a given magnitude/orientation field. */
int ef_nms_f64(const double* d_magnitude, const int64_t* d_orientation, int32_t height, int32_t width,
               double* d_thinned, void* stream);
/* double_threshold (hysteresis.py:54-60) on a given thinned field. */
int ef_double_threshold_f64(const double* d_thinned, int64_t n, double low, double high, uint8_t* d_labels,
                            void* stream);
/* quantize_orientation_array (gradient.py:37-44): int64 degrees. */
int ef_quantize_f64(const double* d_gx, const double* d_gy, int64_t n, int64_t* d_orientation, void* stream);
/* laplacian (gradient.py:96-107): 5-point Laplacian, replicate borders. */
int ef_laplacian_f64(const double* d_src, int32_t height, int32_t width, double* d_out, void* stream);

/* Host-buffer entry point (the e2e path a drop-in user calls): copies u8 frames
 * from h_src to the device, runs ef_canny_u8, and copies labels/final back,
 * overlapping copies and compute across frame chunks on internal streams.
 * Pinned host buffers give full PCIe bandwidth.  Synchronous on return.
 * h_labels may be NULL (edges only -- what the CLI's detect path and
 * edges_to_image, bench.py:129-133, consume): the edge map then crosses PCIe
 * at 1 bit per pixel instead of 2 and only h_final is written. */
int ef_canny_u8_host(const uint8_t* h_src, int64_t batch, int32_t height, int32_t width,
                     const double* h_weights, int32_t radius, double low, double high,
                     uint8_t* h_labels, uint8_t* h_final, int32_t device);

/* Host helper for the drop-in's integer test (GrayImage holds float64,
 * image.py:23-50; the u8 fast path applies when every pixel is an integer in
 * [0,255]): converts n float64 pixels to u8 with the host thread pool.
 * Returns 1 when every value was such an integer (dst complete), 0 when not
 * (dst unspecified), EF_EINVAL on bad arguments.  No device involved. */
int ef_host_f64_to_u8(const double* src, int64_t n, uint8_t* dst);

/* ---- Row-band partition of one huge frame (multi-GPU, trace_edges_parallel
 * hysteresis.py:90-131 generalised across devices). -----------------------
 *
 * A band owns rows [row0, row0+rows) of a frame of full_height rows.  d_src
 * holds rows [row0-halo_top, row0+rows+halo_bot) where
 * halo_top = min(row0, radius+2) and halo_bot = min(full_height-row0-rows, radius+2):
 * neighbours' rows arrive by P2P/NCCL, the frame edge is clamped. */
int ef_band_halo_rows(int32_t radius);

/* Labels of the band plus the band-local hysteresis (tiles, union-find),
 * leaving components that touch the band's top/bottom edge undecided. */
int ef_band_canny_u8(const uint8_t* d_src, int32_t row0, int32_t rows, int32_t full_height,
                     int32_t width, const double* h_weights, int32_t radius, double low,
                     double high, uint8_t* d_labels, uint8_t* d_final, void* d_workspace,
                     size_t workspace_bytes, void* stream);

/* The same with the halo rows read IN PLACE from the neighbour bands (no
 * exchange step): d_band holds this band's `rows` rows only; d_top points at
 * the top_rows = min(row0, radius+2) frame rows just above the band (the last
 * rows of the band above -- on another GPU, a peer pointer from ef_ipc_open,
 * read over NVLink), d_bot at the bot_rows = min(full_height-row0-rows,
 * radius+2) rows just below.  Needs width % 4 == 0 and radius <= 6.  Results
 * equal ef_band_canny_u8 on the contiguous haloed buffer. */
int ef_band_canny_u8_peer(const uint8_t* d_band, const uint8_t* d_top, int32_t top_rows, const uint8_t* d_bot,
                          int32_t bot_rows, int32_t row0, int32_t rows, int32_t full_height, int32_t width,
                          const double* h_weights, int32_t radius, double low, double high, uint8_t* d_labels,
                          uint8_t* d_final, void* d_workspace, size_t workspace_bytes, void* stream);

/* CUDA IPC for the peer halos: export a device pointer (any address inside an
 * allocation) as a 64-byte handle + offset; another process opens it (peer
 * access enabled lazily) and gets a device pointer to the same bytes;
 * ef_ipc_close releases the mapping (pass the base from ef_ipc_open). */
int ef_ipc_export(const void* d_ptr, void* h_handle64, uint64_t* h_offset);
int ef_ipc_open(const void* h_handle64, uint64_t offset, void** d_ptr_out, void** d_base_out);
int ef_ipc_close(void* d_base);


/* Band-local hysteresis only, for labels already computed (the per-band
 * labelling of trace_edges_parallel, hysteresis.py:97-101). */
int ef_band_trace(const uint8_t* d_labels, int32_t rows, int32_t width, uint8_t* d_final, void* d_workspace,
                  size_t workspace_bytes, void* stream);

/* Export the band's two edge rows: for each column of the top and bottom row,
 * the band-local component id (int64, -1 for background) and whether that
 * component is already known to hold a strong pixel (u8).  Arrays have
 * 2*width entries: [0,width) top row, [width,2*width) bottom row. */
int ef_band_edges(const void* d_workspace, size_t workspace_bytes, int32_t rows, int32_t width,
                  int64_t* d_ids, uint8_t* d_strong, void* stream);

/* Host-side cross-band merge (the union-find of hysteresis.py:112-130): given
 * every band's edge rows in band order (nbands blocks of 2*width entries, ids
 * already made globally unique), decide which ids end up connected to a strong
 * pixel.  Writes h_strong_out (same layout as the inputs). */
int ef_band_merge(int32_t nbands, int32_t width, const int64_t* h_ids, const uint8_t* h_strong,
                  uint8_t* h_strong_out);

/* The same merge on the device, stream-ordered (no host round trip): every
 * rank all_gathers the bands' ef_band_edges rows into one device array and
 * runs this on it, reaching the identical decision.  Ids are band-LOCAL here
 * (as ef_band_edges writes them; band k's block is made unique internally as
 * k << 40 | id).  d_scratch: ef_band_merge_scratch_bytes(nbands, width) bytes.
 * Output equals ef_band_merge on the globalised ids. */
size_t ef_band_merge_scratch_bytes(int32_t nbands, int32_t width);
int ef_band_merge_device(int32_t nbands, int32_t width, const int64_t* d_ids, const uint8_t* d_strong,
                         uint8_t* d_strong_out, void* d_scratch, size_t scratch_bytes, void* stream);

/* Apply the merged decision for this band's edge rows and finalise d_final. */
int ef_band_finalize(const uint8_t* d_strong_edges, int32_t rows, int32_t width,
                     const uint8_t* d_labels, uint8_t* d_final, void* d_workspace,
                     size_t workspace_bytes, void* stream);

/* ---- PGM ingest / egress (image.py:87-135; the CLI detect path cli.py:82-90).
 * Host parsing and decoding straight to u8 (no float64 image); errors return
 * EF_EINVAL with the reference's PgmFormatError message in
 * ef_pgm_last_error() and its byte offset in *err_offset. */
typedef struct ef_pgm_info {
    int32_t width, height, maxval;
    int32_t binary;          /* 1: P5 (payload_offset = first payload byte), 0: P2 */
    int64_t payload_offset;  /* P2: where the pixel tokens start */
} ef_pgm_info;

const char* ef_pgm_last_error(void);
/* Parse the header (magic, width, height, maxval; P5: the payload length). */
int ef_pgm_parse(const uint8_t* data, size_t n, ef_pgm_info* info, int64_t* err_offset);
/* Decode the width*height pixels into h_dst (host memory, e.g. pinned) and
 * check them against maxval. */
int ef_pgm_decode_u8(const uint8_t* data, size_t n, const ef_pgm_info* info, uint8_t* h_dst, int64_t* err_offset);
/* "P5\n<w> <h>\n255\n" into h_out; returns its length (or EF_EINVAL). */
int ef_pgm_header(int32_t width, int32_t height, char* h_out, size_t cap);
/* P5 payload of an edge map on the device: 255 where d_final != 0, else 0
 * (save_pgm(edges_to_image(edges)), bench.py:129-133 + image.py:125-135). */
int ef_pgm_encode_edges(const uint8_t* d_final, int64_t n, uint8_t* d_payload, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EDGEFORGE_B200_H */
