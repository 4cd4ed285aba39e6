/*
 * ef_oracle.c -- CPU ORACLE (test infrastructure only; never the product path).
 *
 * A plain-C, scalar, float64 restatement of the reference Canny path
 * (edgeforge, /root/reference/pkg/src/edgeforge) in the reference's exact
 * operation order, so that it reproduces the reference's float64 results
 * bit-for-bit.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library, and only as the
 * checker / the timed CPU baseline.
 *
 * Compile with -ffp-contract=off: the reference evaluates every product and
 * every sum as a separate, correctly rounded numpy ufunc (no FMA).
 *
 * Reference order followed (file:line relative to /root/reference/pkg/src/edgeforge):
 *   horizontal pass  filtering.py:43-55  out = w0*p[x-r]; out += w_i*p[x-r+i]  (edge pad :51)
 *   vertical pass    filtering.py:58-63  out = w0*h[y-r]; out = out + w_i*h[y-r+i] (edge pad :82)
 *   sobel            gradient.py:51-70,73-90  acc starts at +0.0, zero taps skipped,
 *                    gx row-major tap order, gy column-major tap order (:63-65),
 *                    magnitude sqrt(gx*gx+gy*gy) (:82), orientation (:37-44)
 *   nms              nms.py:28-55  keep iff c>=n1 && c>=n2 along the bin, else 0.0
 *   double threshold hysteresis.py:54-60  2 if m>=high, 1 if m>=low, else 0
 *   trace            hysteresis.py:63-69  8-connected components that hold a strong pixel
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define EF_ORACLE_ABI 1

static inline int64_t clampi(int64_t v, int64_t lo, int64_t hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

/* numpy float remainder (npy_divmod): result takes the sign of the divisor. */
static double py_mod(double a, double b) {
    double mod = fmod(a, b);
    if (mod != 0.0) {
        if ((b < 0) != (mod < 0)) mod += b;
    } else {
        mod = copysign(0.0, b);
    }
    return mod;
}

/* gradient.py:37-44 quantize_orientation_array: degrees(arctan2(gy,gx)) % 180,
 * floor((deg+22.5)/45) % 4, times 45.  np.degrees(x) == x * (180/pi). */
int64_t ef_oracle_quantize(double gx, double gy) {
    double deg = atan2(gy, gx) * (180.0 / 3.14159265358979323846);
    deg = py_mod(deg, 180.0);
    double q = floor((deg + 22.5) / 45.0);
    int64_t b = (int64_t)q;
    b = ((b % 4) + 4) % 4;
    return b * 45;
}

/* filtering.py:43-55 -- one row of the horizontal pass, replicate borders. */
static void h_row(const double* src, int64_t W, const double* w, int r, double* out) {
    for (int64_t x = 0; x < W; ++x) {
        double acc = w[0] * src[clampi(x - r, 0, W - 1)];
        for (int i = 1; i <= 2 * r; ++i) {
            double t = w[i] * src[clampi(x - r + i, 0, W - 1)];
            acc = acc + t;
        }
        out[x] = acc;
    }
}

/* gradient.py:51-70 -- 3x3 Sobel taps in reference order on rows (up, mid, dn),
 * each already clamped; column access clamped here. */
static void sobel_row(const double* up, const double* mid, const double* dn, int64_t W,
                      double* gx, double* gy, double* mag, int64_t* ori) {
    for (int64_t x = 0; x < W; ++x) {
        int64_t xl = clampi(x - 1, 0, W - 1), xr = clampi(x + 1, 0, W - 1);
        /* SOBEL_X row-major: (0,0)-1 (0,2)+1 (1,0)-2 (1,2)+2 (2,0)-1 (2,2)+1 */
        double a = 0.0;
        a = a + (-1.0 * up[xl]);
        a = a + (1.0 * up[xr]);
        a = a + (-2.0 * mid[xl]);
        a = a + (2.0 * mid[xr]);
        a = a + (-1.0 * dn[xl]);
        a = a + (1.0 * dn[xr]);
        /* SOBEL_Y column-major: (0,0)-1 (2,0)+1 (0,1)-2 (2,1)+2 (0,2)-1 (2,2)+1 */
        double b = 0.0;
        b = b + (-1.0 * up[xl]);
        b = b + (1.0 * dn[xl]);
        b = b + (-2.0 * up[x]);
        b = b + (2.0 * dn[x]);
        b = b + (-1.0 * up[xr]);
        b = b + (1.0 * dn[xr]);
        double m2a = a * a, m2b = b * b;
        double m = sqrt(m2a + m2b);
        if (gx) gx[x] = a;
        if (gy) gy[x] = b;
        mag[x] = m;
        ori[x] = ef_oracle_quantize(a, b);
    }
}

/* nms.py:28-33 neighbour offsets (dy, dx) per bin. */
static const int NB[4][2][2] = {
    {{0, -1}, {0, 1}},   /* 0   : left / right          */
    {{-1, 1}, {1, -1}},  /* 45  : up-right / down-left  */
    {{-1, 0}, {1, 0}},   /* 90  : up / down             */
    {{-1, -1}, {1, 1}},  /* 135 : up-left / down-right  */
};

static inline uint8_t classify(double v, double low, double high) {
    return v >= high ? 2 : (v >= low ? 1 : 0); /* hysteresis.py:57-59 */
}

/* --------------------------------------------------------------------------
 * Full-frame stage dump (small images): every intermediate array.
 * blurred/gx/gy/mag/thin are HxW float64, ori is HxW int64, labels u8, final u8.
 * Any output pointer may be NULL except the ones later stages need internally.
 * ------------------------------------------------------------------------ */
int ef_oracle_stages(const double* px, int64_t H, int64_t W, const double* w, int r,
                     double low, double high, double* blurred, double* gx, double* gy,
                     double* mag, int64_t* ori, double* thin, uint8_t* labels) {
    if (H < 1 || W < 1 || r < 0) return -1;
    size_t n = (size_t)H * (size_t)W;
    double* h = (double*)malloc(n * sizeof(double));
    double* b = blurred ? blurred : (double*)malloc(n * sizeof(double));
    double* m = mag ? mag : (double*)malloc(n * sizeof(double));
    int64_t* o = ori ? ori : (int64_t*)malloc(n * sizeof(int64_t));
    if (!h || !b || !m || !o) return -2;
    for (int64_t y = 0; y < H; ++y) h_row(px + y * W, W, w, r, h + y * W);
    /* filtering.py:58-63,82 vertical pass */
    for (int64_t y = 0; y < H; ++y) {
        for (int64_t x = 0; x < W; ++x) {
            double acc = w[0] * h[clampi(y - r, 0, H - 1) * W + x];
            for (int i = 1; i <= 2 * r; ++i) {
                double t = w[i] * h[clampi(y - r + i, 0, H - 1) * W + x];
                acc = acc + t;
            }
            b[y * W + x] = acc;
        }
    }
    for (int64_t y = 0; y < H; ++y) {
        const double* up = b + clampi(y - 1, 0, H - 1) * W;
        const double* dn = b + clampi(y + 1, 0, H - 1) * W;
        sobel_row(up, b + y * W, dn, W, gx ? gx + y * W : NULL, gy ? gy + y * W : NULL,
                  m + y * W, o + y * W);
    }
    for (int64_t y = 0; y < H; ++y) {
        for (int64_t x = 0; x < W; ++x) {
            int k = (int)(o[y * W + x] / 45);
            double c = m[y * W + x];
            double n1 = m[clampi(y + NB[k][0][0], 0, H - 1) * W + clampi(x + NB[k][0][1], 0, W - 1)];
            double n2 = m[clampi(y + NB[k][1][0], 0, H - 1) * W + clampi(x + NB[k][1][1], 0, W - 1)];
            double t = (c >= n1 && c >= n2) ? c : 0.0;
            if (thin) thin[y * W + x] = t;
            if (labels) labels[y * W + x] = classify(t, low, high);
        }
    }
    free(h);
    if (!blurred) free(b);
    if (!mag) free(m);
    if (!ori) free(o);
    return 0;
}

/* --------------------------------------------------------------------------
 * Banded, memory-lean labels for large images / batches (same arithmetic).
 * Computes labels for rows [y0, y1) of one HxW frame.
 * ------------------------------------------------------------------------ */
static int band_labels(const double* px, const uint8_t* px8, int64_t H, int64_t W,
                       const double* w, int r, double low, double high, int64_t y0,
                       int64_t y1, uint8_t* labels) {
    int64_t hb0 = clampi(y0 - 2 - r, 0, H - 1), hb1 = clampi(y1 + 1 + r, 0, H - 1);
    int64_t bb0 = clampi(y0 - 2, 0, H - 1), bb1 = clampi(y1 + 1, 0, H - 1);
    int64_t mb0 = clampi(y0 - 1, 0, H - 1), mb1 = clampi(y1, 0, H - 1);
    int64_t nh = hb1 - hb0 + 1, nbr = bb1 - bb0 + 1, nm = mb1 - mb0 + 1;
    double* h = (double*)malloc((size_t)nh * W * sizeof(double));
    double* b = (double*)malloc((size_t)nbr * W * sizeof(double));
    double* m = (double*)malloc((size_t)nm * W * sizeof(double));
    int64_t* o = (int64_t*)malloc((size_t)nm * W * sizeof(int64_t));
    double* row = (double*)malloc((size_t)W * sizeof(double));
    if (!h || !b || !m || !o || !row) return -2;
    for (int64_t y = hb0; y <= hb1; ++y) {
        const double* src = px ? px + y * W : row;
        if (!px)
            for (int64_t x = 0; x < W; ++x) row[x] = (double)px8[y * W + x];
        h_row(src, W, w, r, h + (y - hb0) * W);
    }
    for (int64_t y = bb0; y <= bb1; ++y) {
        for (int64_t x = 0; x < W; ++x) {
            double acc = w[0] * h[(clampi(y - r, 0, H - 1) - hb0) * W + x];
            for (int i = 1; i <= 2 * r; ++i) {
                double t = w[i] * h[(clampi(y - r + i, 0, H - 1) - hb0) * W + x];
                acc = acc + t;
            }
            b[(y - bb0) * W + x] = acc;
        }
    }
    for (int64_t y = mb0; y <= mb1; ++y) {
        const double* up = b + (clampi(y - 1, 0, H - 1) - bb0) * W;
        const double* dn = b + (clampi(y + 1, 0, H - 1) - bb0) * W;
        sobel_row(up, b + (y - bb0) * W, dn, W, NULL, NULL, m + (y - mb0) * W, o + (y - mb0) * W);
    }
    for (int64_t y = y0; y < y1; ++y) {
        for (int64_t x = 0; x < W; ++x) {
            int k = (int)(o[(y - mb0) * W + x] / 45);
            double c = m[(y - mb0) * W + x];
            double n1 = m[(clampi(y + NB[k][0][0], 0, H - 1) - mb0) * W + clampi(x + NB[k][0][1], 0, W - 1)];
            double n2 = m[(clampi(y + NB[k][1][0], 0, H - 1) - mb0) * W + clampi(x + NB[k][1][1], 0, W - 1)];
            double t = (c >= n1 && c >= n2) ? c : 0.0;
            labels[y * W + x] = classify(t, low, high);
        }
    }
    free(h); free(b); free(m); free(o); free(row);
    return 0;
}

/* hysteresis.py:63-69 -- keep 8-connected components of labels!=0 that hold a
 * strong pixel.  Flood fill from every strong seed (explicit stack). */
int ef_oracle_trace(const uint8_t* labels, int64_t H, int64_t W, uint8_t* final_out) {
    size_t n = (size_t)H * (size_t)W;
    memset(final_out, 0, n);
    size_t cap = 1 << 16, top = 0;
    int64_t* stack = (int64_t*)malloc(cap * sizeof(int64_t));
    if (!stack) return -2;
    for (size_t i = 0; i < n; ++i) {
        if (labels[i] != 2 || final_out[i]) continue;
        final_out[i] = 1;
        stack[top++] = (int64_t)i;
        while (top) {
            int64_t p = stack[--top];
            int64_t y = p / W, x = p % W;
            for (int dy = -1; dy <= 1; ++dy) {
                int64_t ny = y + dy;
                if (ny < 0 || ny >= H) continue;
                for (int dx = -1; dx <= 1; ++dx) {
                    int64_t nx = x + dx;
                    if (nx < 0 || nx >= W) continue;
                    int64_t q = ny * W + nx;
                    if (labels[q] != 0 && !final_out[q]) {
                        final_out[q] = 1;
                        if (top == cap) {
                            cap *= 2;
                            int64_t* s2 = (int64_t*)realloc(stack, cap * sizeof(int64_t));
                            if (!s2) { free(stack); return -2; }
                            stack = s2;
                        }
                        stack[top++] = q;
                    }
                }
            }
        }
    }
    free(stack);
    return 0;
}

/* Work item fan-out over plain pthreads (an atomic task counter). */
typedef struct {
    const double* px; const uint8_t* px8; int64_t H, W; const double* w; int r;
    double low, high; uint8_t* labels; uint8_t* final_out; int64_t band_rows, nbands, total;
    int64_t next; int err; int phase; pthread_mutex_t mu;
} pool_t;

static void* pool_worker(void* arg) {
    pool_t* p = (pool_t*)arg;
    for (;;) {
        pthread_mutex_lock(&p->mu);
        int64_t t = p->next++;
        pthread_mutex_unlock(&p->mu);
        if (t >= p->total) break;
        int e;
        if (p->phase == 0) {
            int64_t f = t / p->nbands, bi = t % p->nbands;
            int64_t y0 = bi * p->band_rows;
            int64_t y1 = y0 + p->band_rows < p->H ? y0 + p->band_rows : p->H;
            size_t off = (size_t)f * p->H * p->W;
            e = band_labels(p->px ? p->px + off : NULL, p->px ? NULL : p->px8 + off, p->H, p->W,
                            p->w, p->r, p->low, p->high, y0, y1, p->labels + off);
        } else {
            size_t off = (size_t)t * p->H * p->W;
            e = ef_oracle_trace(p->labels + off, p->H, p->W, p->final_out + off);
        }
        if (e) {
            pthread_mutex_lock(&p->mu);
            p->err = e;
            pthread_mutex_unlock(&p->mu);
        }
    }
    return NULL;
}

static int run_pool(pool_t* p, int threads) {
    if (threads < 1) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    int started = 0;
    for (int i = 1; i < threads; ++i)
        if (pthread_create(&tid[started], NULL, pool_worker, p) == 0) ++started;
    pool_worker(p);
    for (int i = 0; i < started; ++i) pthread_join(tid[i], NULL);
    return p->err;
}

/* run_pipeline (bench.py:61-126, canny operator, explicit thresholds) over a
 * batch of frames.  Input either float64 (px) or u8 (px8); one must be NULL.
 * Stencil stages run banded over `threads` pthreads (bands are independent:
 * every clamp is against the full frame); tracing is serial per frame, like
 * the reference's default serial hysteresis (frames trace in parallel). */
int ef_oracle_canny(const double* px, const uint8_t* px8, int64_t batch, int64_t H, int64_t W,
                    const double* w, int r, double low, double high, uint8_t* labels,
                    uint8_t* final_out, int threads, int64_t band_rows) {
    if (H < 1 || W < 1 || batch < 1 || r < 0) return -1;
    if (band_rows < 1) band_rows = 64;
    pool_t p;
    memset(&p, 0, sizeof p);
    p.px = px; p.px8 = px8; p.H = H; p.W = W; p.w = w; p.r = r; p.low = low; p.high = high;
    p.labels = labels; p.final_out = final_out; p.band_rows = band_rows;
    p.nbands = (H + band_rows - 1) / band_rows;
    p.total = batch * p.nbands;
    pthread_mutex_init(&p.mu, NULL);
    int err = run_pool(&p, threads);
    if (!err && final_out) {
        p.phase = 1; p.next = 0; p.total = batch;
        err = run_pool(&p, threads);
    }
    pthread_mutex_destroy(&p.mu);
    return err ? -2 : 0;
}

int ef_oracle_abi(void) { return EF_ORACLE_ABI; }
