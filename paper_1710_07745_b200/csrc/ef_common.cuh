// ef_common.cuh -- shared device code for the B200 Canny path.
//
// Two arithmetic regimes live side by side:
//  * EXACT: float64 in the reference's operation order, every product and sum
//    separately rounded (__dmul_rn / __dadd_rn forbid FMA contraction), so a
//    value equals the numpy reference bit-for-bit.  Used for float64 inputs,
//    intermediates, auto-threshold max and for fix-ups of uncertified pixels.
//  * FAST: fp32 with folded symmetric taps and FMAs, plus certified error
//    bounds (FastParams) that say when an fp32 decision provably equals the
//    exact one.  Used by the fused classify kernel on u8 inputs.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/edgeforge_b200.h"

namespace ef {

constexpr int kMaxR = EF_MAX_RADIUS;
constexpr uint8_t kFlag = 0x80;  // label byte marker: decision not certified yet

// Debug build (-DEF_DEBUG_CHECKS, tools/gpu_debug_checks.sh): device-side bounds
// assertions on the shared-memory and global indices of the kernels, the
// substitute for compute-sanitizer, which is closed on this GPU pool.  A failed
// check traps the kernel (the call returns EF_ECUDA).  Compiled out otherwise.
#ifdef EF_DEBUG_CHECKS
#define EF_DCHECK(cond)                                                                           \
    do {                                                                                          \
        if (!(cond)) {                                                                            \
            printf("EF_DCHECK failed: %s (%s:%d) block (%d,%d,%d) thread %d\n", #cond, __FILE__, \
                   __LINE__, (int)blockIdx.x, (int)blockIdx.y, (int)blockIdx.z, (int)threadIdx.x); \
            __trap();                                                                             \
        }                                                                                         \
    } while (0)
#else
#define EF_DCHECK(cond) ((void)0)
#endif

// Reference label values (hysteresis.py:19-21).
constexpr uint8_t kNone = 0, kWeak = 1, kStrong = 2;

struct ExactParams {
    double w[2 * kMaxR + 1];  // GaussianKernel.weights, left to right
    int r;
    double low, high;  // Thresholds (hysteresis.py:26-33)
};

struct FastParams {
    float wf[kMaxR + 1];  // folded: wf[0] = centre weight, wf[k] = weight at +-k
    int r;
    // certified comparisons of the fp32 magnitude m against the thresholds:
    // m < lo_lo -> certainly below low, m > lo_hi -> certainly >= low, else flag
    float lo_lo, lo_hi, hi_lo, hi_hi;
    float e_nms;  // |c - n| > e_nms -> the NMS comparison is certain (any magnitudes up to 1443)
    // magnitude-relative form used by the production classifier: certain iff
    // |c - n| > e_nms0 + e_nms_rel * (c + n)
    float e_nms0, e_nms_rel;
    float e_sec;  // |t*a - b| > e_sec -> the orientation sector is certain
    int cls0;     // class of a suppressed pixel (thinned value 0.0)
    int no_v2;    // a caller buffer is not 4-byte aligned: the generic byte-wise classifier only
};

// Workspace header (device memory, start of the caller's workspace).
struct WsHeader {
    ef_stats stats;          // accumulated counters
    unsigned long long fix_count;
    unsigned long long fix_cap;
    unsigned int overflow;           // fix list overflowed: fix-up kernel scans all pixels
    unsigned int plist_overflow;     // a pending-list stripe overflowed: H4 re-runs tile CCL
    unsigned int dense_count;        // tiles H1's warp kernel handed to the block kernel
    unsigned int node_overflow;      // a node-list stripe overflowed: H3 scans every perimeter slot
    unsigned int pad[4];
};

__host__ __device__ inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// numpy float remainder (npy_divmod): sign of the divisor.
__device__ inline double py_mod(double a, double b) {
    double m = fmod(a, b);
    if (m != 0.0) {
        if ((b < 0) != (m < 0)) m = __dadd_rn(m, b);
    } else {
        m = copysign(0.0, b);
    }
    return m;
}

// Orientation bin 0..3 (0, 45, 90, 135 degrees) of an exact float64 gradient,
// equal to quantize_orientation_array (gradient.py:37-44).
//
// The reference computes degrees(arctan2(gy,gx)) % 180 and floors
// (deg + 22.5)/45.  Away from the four sector boundaries that equals a purely
// geometric test -- |gy| < tan(22.5)|gx| is bin 0, |gx| < tan(22.5)|gy| is bin
// 2, otherwise 45 if gx*gy > 0 else 135 -- which needs no transcendental.  The
// boundaries are irrational slopes, so a float64 gradient lands within 1e-12
// (relative) of one essentially never; if it does, the reference's own formula
// is evaluated with CUDA's atan2 and the pixel is counted as ambiguous.
__device__ inline int exact_sector(double gx, double gy, unsigned long long* ambiguous) {
    const double t = 0.41421356237309503;  // nearest double to sqrt(2) - 1
    double a = fabs(gx), b = fabs(gy);
    double u = __dadd_rn(__dmul_rn(t, a), -b);  // > 0 : bin 0
    double v = __dadd_rn(__dmul_rn(t, b), -a);  // > 0 : bin 2
    double tol = 1e-12 * (a + b);
    if ((fabs(u) <= tol || fabs(v) <= tol) && (a + b) > 0.0) {
        if (ambiguous) atomicAdd(ambiguous, 1ull);
        double deg = __dmul_rn(atan2(gy, gx), 180.0 / 3.14159265358979323846);
        deg = py_mod(deg, 180.0);
        long long q = (long long)floor(__ddiv_rn(__dadd_rn(deg, 22.5), 45.0));
        return (int)(((q % 4) + 4) % 4);
    }
    if (a == 0.0 && b == 0.0) return 0;  // arctan2(0, 0) = 0
    if (u > 0.0) return 0;
    if (v > 0.0) return 2;
    return ((gx > 0.0) == (gy > 0.0)) ? 1 : 3;
}

// nms.py:28-33 neighbour offsets (dy, dx) per bin.
// bin 0: left/right, 1 (45): up-right/down-left, 2 (90): up/down, 3 (135): up-left/down-right.
__host__ __device__ inline void nb_offsets(int s, int& dy1, int& dx1, int& dy2, int& dx2) {
    dy1 = s == 0 ? 0 : -1;
    dy2 = -dy1;
    dx1 = s == 0 ? -1 : (s == 1 ? 1 : (s == 2 ? 0 : -1));
    dx2 = -dx1;
}

__device__ inline uint8_t classify_exact(double v, double low, double high) {
    return v >= high ? kStrong : (v >= low ? kWeak : kNone);  // hysteresis.py:57-59
}

// Exact Sobel at one position from a 3x3 block of blurred values
// (gradient.py:51-70): acc starts at +0.0, zero taps skipped, gx in row-major
// tap order, gy in column-major tap order.  b[dy][dx], dy/dx in 0..2.
__device__ inline void exact_sobel(const double b[3][3], double& gx, double& gy) {
    double a = 0.0;
    a = __dadd_rn(a, -b[0][0]);
    a = __dadd_rn(a, b[0][2]);
    a = __dadd_rn(a, __dmul_rn(-2.0, b[1][0]));
    a = __dadd_rn(a, __dmul_rn(2.0, b[1][2]));
    a = __dadd_rn(a, -b[2][0]);
    a = __dadd_rn(a, b[2][2]);
    double c = 0.0;
    c = __dadd_rn(c, -b[0][0]);
    c = __dadd_rn(c, b[2][0]);
    c = __dadd_rn(c, __dmul_rn(-2.0, b[0][1]));
    c = __dadd_rn(c, __dmul_rn(2.0, b[2][1]));
    c = __dadd_rn(c, -b[0][2]);
    c = __dadd_rn(c, b[2][2]);
    gx = a;
    gy = c;
}

__device__ inline double exact_mag(double gx, double gy) {
    return __dsqrt_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)));  // gradient.py:82
}

template <typename T>
__device__ inline double load_px(const T* p) { return (double)*p; }

}  // namespace ef
