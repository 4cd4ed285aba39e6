// ef_host.cu -- host side of the host-buffer entry point (ef_canny_u8_host).
//
// The reference's run_pipeline returns host arrays (EdgeMap.labels u8 and
// EdgeMap.final bool, pkg/src/edgeforge/hysteresis.py:36-51), so the drop-in
// pays PCIe both ways.  Three things keep the transfer at the input's PCIe
// cost instead of input + 2 B/px of output:
//   * a device pack kernel folds (labels, final) into 2 bits per pixel -- final
//     is implied for strong pixels and impossible for background ones, so the
//     four states {0/F, 1/F, 1/T, 2/T} are the whole output (0.25 B/px D2H);
//   * a pool of host threads expands the packed stream into the caller's two
//     arrays with non-temporal stores (no read-for-ownership, pageable or not);
//   * pageable inputs are staged into pinned memory by the same pool, so the
//     DMA always runs from pinned pages.
#if defined(__x86_64__) && !defined(EF_PORTABLE_HOST)
#define EF_X86 1
#include <emmintrin.h>
#include <immintrin.h>
#include <cpuid.h>
#else
#define EF_X86 0  // aarch64 (Grace): scalar unpack, plain copies, no cache-line eviction
#endif
#include <sched.h>
#ifdef __linux__
#include <sys/prctl.h>
#endif

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "ef_host.h"

namespace ef {

// --------------------------------------------------------------- device ----
// code = 0 (label 0), 1 (weak, not final), 2 (weak, final), 3 (strong)
__device__ __forceinline__ uint32_t pack_code(uint32_t lab, uint32_t fin) {
    return lab == 0u ? 0u : (lab >= 2u ? 3u : (fin ? 2u : 1u));
}

__global__ void pack_kernel(const uint8_t* __restrict__ labels, const uint8_t* __restrict__ final_map, long long n,
                            uint8_t* __restrict__ packed) {
    const long long nq = (n + 15) / 16;  // 16 pixels -> 4 packed bytes per thread
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (long long)gridDim.x * blockDim.x) {
        const long long p0 = q * 16;
        uint32_t out = 0;
        if (p0 + 16 <= n) {
            const uint4 l = *reinterpret_cast<const uint4*>(labels + p0);
            const uint4 f = *reinterpret_cast<const uint4*>(final_map + p0);
            const uint32_t lw[4] = {l.x, l.y, l.z, l.w}, fw[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
            for (int k = 0; k < 16; ++k)
                out |= pack_code((lw[k >> 2] >> (8 * (k & 3))) & 0xffu, (fw[k >> 2] >> (8 * (k & 3))) & 0xffu)
                       << (2 * k);
        } else {
            for (int k = 0; p0 + k < n; ++k) out |= pack_code(labels[p0 + k], final_map[p0 + k]) << (2 * k);
        }
        const long long nb = min(4ll, (n - p0 + 3) / 4);  // packed bytes this thread owns
        if (nb == 4) *reinterpret_cast<uint32_t*>(packed + 4 * q) = out;
        else
            for (int b = 0; b < nb; ++b) packed[4 * q + b] = (uint8_t)(out >> (8 * b));
    }
}

cudaError_t launch_pack(const uint8_t* labels, const uint8_t* final_map, long long n, uint8_t* packed, int sm_count,
                        cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const long long nq = (n + 15) / 16;
    const int threads = 256;
    const long long want = (nq + threads - 1) / threads;
    const int blocks = (int)std::min<long long>(want, (long long)sm_count * 8);
    pack_kernel<<<blocks, threads, 0, st>>>(labels, final_map, n, packed);
    return cudaGetLastError();
}

// Edges-only calls (h_labels == NULL): the final map alone, 1 bit per pixel
// (bit k of byte j = pixel 8 j + k).  32 pixels -> 4 packed bytes per thread.
__global__ void pack_final_kernel(const uint8_t* __restrict__ final_map, long long n, uint8_t* __restrict__ packed) {
    const long long nq = (n + 31) / 32;
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (long long)gridDim.x * blockDim.x) {
        const long long p0 = q * 32;
        uint32_t out = 0;
        if (p0 + 32 <= n) {
            const uint4 a = *reinterpret_cast<const uint4*>(final_map + p0);
            const uint4 b = *reinterpret_cast<const uint4*>(final_map + p0 + 16);
            const uint32_t fw[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int k = 0; k < 8; ++k)  // bytes are 0 / 1: gather the four low bits of a word into a nibble
                out |= (((fw[k] & 0x01010101u) * 0x10204080u) >> 28) << (4 * k);
        } else {
            for (int k = 0; p0 + k < n; ++k) out |= (uint32_t)(final_map[p0 + k] & 1u) << k;
        }
        const long long nb = min(4ll, (n - p0 + 7) / 8);  // packed bytes this thread owns
        if (nb == 4) *reinterpret_cast<uint32_t*>(packed + 4 * q) = out;
        else
            for (int b = 0; b < nb; ++b) packed[4 * q + b] = (uint8_t)(out >> (8 * b));
    }
}

cudaError_t launch_pack_final(const uint8_t* final_map, long long n, uint8_t* packed, int sm_count, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const long long nq = (n + 31) / 32;
    const int threads = 256;
    const long long want = (nq + threads - 1) / threads;
    const int blocks = (int)std::min<long long>(want, (long long)sm_count * 8);
    pack_final_kernel<<<blocks, threads, 0, st>>>(final_map, n, packed);
    return cudaGetLastError();
}

// ----------------------------------------------------------------- host ----
namespace {
struct Luts {
    uint32_t lab[256], fin[256];
    Luts() {
        for (int b = 0; b < 256; ++b) {
            uint32_t l = 0, f = 0;
            for (int k = 0; k < 4; ++k) {
                const int c = (b >> (2 * k)) & 3;
                l |= (uint32_t)(c == 0 ? 0 : (c == 3 ? 2 : 1)) << (8 * k);
                f |= (uint32_t)(c >= 2 ? 1 : 0) << (8 * k);
            }
            lab[b] = l;
            fin[b] = f;
        }
    }
};
const Luts& luts() {
    static const Luts L;
    return L;
}
}  // namespace

// Evict the packed staging lines after the unpack has read them: the next
// D2H into lines still held by the CPU caches runs several times slower.
#if EF_X86
__attribute__((target("clflushopt"))) static void flush_opt(const uint8_t* p, size_t n) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(63);
    for (uintptr_t a = a0; a < reinterpret_cast<uintptr_t>(p) + n; a += 64) _mm_clflushopt((void*)a);
    _mm_sfence();
}

void flush_lines(const uint8_t* p, size_t n) {
    static const bool has_opt = [] {
        unsigned a, b, c, d;
        return __get_cpuid_count(7, 0, &a, &b, &c, &d) && (b & (1u << 23));
    }();
    if (has_opt) {
        flush_opt(p, n);
        return;
    }
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(63);
    for (uintptr_t a = a0; a < reinterpret_cast<uintptr_t>(p) + n; a += 64) _mm_clflush((void*)a);
    _mm_mfence();
}
#else
void flush_lines(const uint8_t*, size_t) {}  // coherent DMA; eviction is an x86 tuning only
#endif

#if EF_X86
// AVX2 + BMI2 body: 8 packed bytes (32 pixels) per step.  pdep spreads each
// 2-bit code into a byte; label = (code + 1) >> 1 and final = code >> 1 bytewise
// (codes <= 3, so no carries cross bytes); two 32-byte non-temporal stores.
// Returns the first packed byte not done; labels + 4*j must be 32-byte aligned.
__attribute__((target("avx2,bmi2"))) static size_t unpack_avx2(const uint8_t* packed, size_t j, size_t end,
                                                                uint8_t* labels, uint8_t* final_map) {
    const __m256i one = _mm256_set1_epi8(1), low7 = _mm256_set1_epi8(0x7f);
    for (; j + 8 <= end; j += 8) {
        uint64_t w;
        std::memcpy(&w, packed + j, 8);
        const __m256i codes = _mm256_setr_epi64x(
            (long long)_pdep_u64(w & 0xffffu, 0x0303030303030303ull),
            (long long)_pdep_u64((w >> 16) & 0xffffu, 0x0303030303030303ull),
            (long long)_pdep_u64((w >> 32) & 0xffffu, 0x0303030303030303ull),
            (long long)_pdep_u64((w >> 48) & 0xffffu, 0x0303030303030303ull));
        const __m256i lab = _mm256_and_si256(_mm256_srli_epi16(_mm256_add_epi8(codes, one), 1), low7);
        const __m256i fin = _mm256_and_si256(_mm256_srli_epi16(codes, 1), one);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(labels + 4 * j), lab);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(final_map + 4 * j), fin);
    }
    return j;
}

static bool has_avx2_bmi2() {
    static const bool ok = __builtin_cpu_supports("avx2") && __builtin_cpu_supports("bmi2");
    return ok;
}
#endif

void unpack_codes(const uint8_t* packed, size_t byte0, size_t byte1, size_t npx, uint8_t* labels,
                  uint8_t* final_map) {
    const Luts& T = luts();
    // pixels 4*byte0 .. min(4*byte1, npx)
    size_t j = byte0;
    const size_t full_end = std::min(byte1, npx / 4);  // bytes whose 4 pixels all exist
    auto scalar = [&](size_t b) {
        const uint32_t l = T.lab[packed[b]], f = T.fin[packed[b]];
        std::memcpy(labels + 4 * b, &l, 4);
        std::memcpy(final_map + 4 * b, &f, 4);
    };
#if EF_X86
    const bool same_phase32 = ((reinterpret_cast<uintptr_t>(labels) ^ reinterpret_cast<uintptr_t>(final_map)) & 31) == 0;
    if (same_phase32 && has_avx2_bmi2()) {
        while (j < full_end && (reinterpret_cast<uintptr_t>(labels + 4 * j) & 31)) scalar(j++);
        j = unpack_avx2(packed, j, full_end, labels, final_map);
        _mm_sfence();
    }
    const bool same_phase = ((reinterpret_cast<uintptr_t>(labels) ^ reinterpret_cast<uintptr_t>(final_map)) & 15) == 0;
    if (same_phase) {
        while (j < full_end && (reinterpret_cast<uintptr_t>(labels + 4 * j) & 15)) scalar(j++);
        for (; j + 4 <= full_end; j += 4) {
            const uint8_t* p = packed + j;
            const __m128i l = _mm_setr_epi32((int)T.lab[p[0]], (int)T.lab[p[1]], (int)T.lab[p[2]], (int)T.lab[p[3]]);
            const __m128i f = _mm_setr_epi32((int)T.fin[p[0]], (int)T.fin[p[1]], (int)T.fin[p[2]], (int)T.fin[p[3]]);
            _mm_stream_si128(reinterpret_cast<__m128i*>(labels + 4 * j), l);
            _mm_stream_si128(reinterpret_cast<__m128i*>(final_map + 4 * j), f);
        }
        _mm_sfence();
    }
#endif
    for (; j < full_end; ++j) scalar(j);
    if (j < byte1 && 4 * j < npx) {  // last partial byte
        const uint32_t l = T.lab[packed[j]], f = T.fin[packed[j]];
        for (size_t k = 0; 4 * j + k < npx; ++k) {
            labels[4 * j + k] = (uint8_t)(l >> (8 * k));
            final_map[4 * j + k] = (uint8_t)(f >> (8 * k));
        }
    }
}

#if EF_X86
// 4 packed bytes (32 pixels) per step: pdep spreads 8 bits into 8 bytes of 0 / 1.
__attribute__((target("avx2,bmi2"))) static size_t unpack_bits_avx2(const uint8_t* packed, size_t j, size_t end,
                                                                     uint8_t* final_map) {
    const uint64_t ones = 0x0101010101010101ull;
    for (; j + 4 <= end; j += 4) {
        uint32_t w;
        std::memcpy(&w, packed + j, 4);
        const __m256i v = _mm256_setr_epi64x((long long)_pdep_u64(w & 0xffu, ones), (long long)_pdep_u64((w >> 8) & 0xffu, ones),
                                             (long long)_pdep_u64((w >> 16) & 0xffu, ones), (long long)_pdep_u64(w >> 24, ones));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(final_map + 8 * j), v);
    }
    return j;
}
#endif

// expand packed bits [byte0, byte1) of an npx-pixel stream into final_map (0 / 1 bytes)
void unpack_bits(const uint8_t* packed, size_t byte0, size_t byte1, size_t npx, uint8_t* final_map) {
    auto scalar = [&](size_t b) {
        uint64_t v = 0;
        for (int k = 0; k < 8; ++k) v |= (uint64_t)((packed[b] >> k) & 1u) << (8 * k);
        std::memcpy(final_map + 8 * b, &v, 8);
    };
    size_t j = byte0;
    const size_t full_end = std::min(byte1, npx / 8);  // bytes whose 8 pixels all exist
#if EF_X86
    if (has_avx2_bmi2()) {
        while (j < full_end && (reinterpret_cast<uintptr_t>(final_map + 8 * j) & 31)) scalar(j++);
        if ((reinterpret_cast<uintptr_t>(final_map + 8 * j) & 31) == 0) j = unpack_bits_avx2(packed, j, full_end, final_map);
        _mm_sfence();
    }
#endif
    for (; j < full_end; ++j) scalar(j);
    if (j < byte1 && 8 * j < npx)  // last partial byte
        for (size_t k = 0; 8 * j + k < npx; ++k) final_map[8 * j + k] = (uint8_t)((packed[j] >> k) & 1u);
}

// Fixed pool of worker threads with a FIFO (front pushes jump the queue).
struct HostPool::Impl {
    std::mutex mu;
    std::condition_variable cv;
    std::deque<std::function<void()>> q;
    std::vector<std::thread> th;
};

HostPool::HostPool(int n) : impl_(new Impl) {
    for (int i = 0; i < n; ++i)
        impl_->th.emplace_back([this] {
#if defined(__linux__) && !defined(EF_NO_TIMERSLACK)
            // the chunk waits sleep-poll in 20 us steps: the default 50 us timer slack would triple them
            prctl(PR_SET_TIMERSLACK, 2000UL, 0UL, 0UL, 0UL);
#endif
            for (;;) {
                std::function<void()> f;
                {
                    std::unique_lock<std::mutex> lk(impl_->mu);
                    impl_->cv.wait(lk, [this] { return !impl_->q.empty(); });
                    f = std::move(impl_->q.front());
                    impl_->q.pop_front();
                }
                f();
            }
        });
    for (auto& t : impl_->th) t.detach();  // the pool lives for the process
}

int HostPool::size() const { return (int)impl_->th.size(); }

void HostPool::submit(std::function<void()> f, bool front) {
    {
        std::lock_guard<std::mutex> lk(impl_->mu);
        if (front) impl_->q.push_front(std::move(f));
        else impl_->q.push_back(std::move(f));
    }
    impl_->cv.notify_one();
}

HostPool& host_pool() {
    static HostPool* pool = [] {
        cpu_set_t set;
        int n = 8;
        if (sched_getaffinity(0, sizeof set, &set) == 0) n = CPU_COUNT(&set);
        // one process per GPU (torchrun): share the host's cores between the
        // local ranks instead of oversubscribing them
        if (const char* lw = getenv("LOCAL_WORLD_SIZE")) n = std::max(1, n / std::max(1, atoi(lw)));
        return new HostPool(std::max(1, std::min(n, 32)));
    }();
    return *pool;
}

void Latch::add(int n) {
    std::lock_guard<std::mutex> lk(mu);
    count += n;
}
void Latch::done() {
    std::lock_guard<std::mutex> lk(mu);
    if (--count == 0) cv.notify_all();
}
void Latch::wait() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [this] { return count == 0; });
}

// copy into pinned staging with non-temporal stores: the DMA that reads the
// staging next must not find its lines dirty in the CPU caches
static void stream_copy(uint8_t* dst, const uint8_t* src, size_t bytes) {
#if !EF_X86
    std::memcpy(dst, src, bytes);
    return;
#else
    size_t i = 0;
    while (i < bytes && (reinterpret_cast<uintptr_t>(dst + i) & 15)) {
        dst[i] = src[i];
        ++i;
    }
    for (; i + 64 <= bytes; i += 64) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
        const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
        const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
    }
    _mm_sfence();
    for (; i < bytes; ++i) dst[i] = src[i];
#endif
}

#if EF_X86
// 8 doubles per step: truncate, convert back and compare (NaN and out-of-range
// values fail the comparison or the range test), pack to bytes with saturation
// (dst is unspecified once a value failed).  Returns the first index not done.
__attribute__((target("avx2"))) static size_t f64_to_u8_avx2(const double* src, size_t n, uint8_t* dst, bool& ok) {
    __m256d bad = _mm256_setzero_pd();
    const __m128i lim = _mm_set1_epi32(255);
    __m128i badi = _mm_setzero_si128();
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        const __m256d a = _mm256_loadu_pd(src + i), b = _mm256_loadu_pd(src + i + 4);
        const __m128i ta = _mm256_cvttpd_epi32(a), tb = _mm256_cvttpd_epi32(b);
        bad = _mm256_or_pd(bad, _mm256_cmp_pd(_mm256_cvtepi32_pd(ta), a, _CMP_NEQ_UQ));
        bad = _mm256_or_pd(bad, _mm256_cmp_pd(_mm256_cvtepi32_pd(tb), b, _CMP_NEQ_UQ));
        // 0 <= t <= 255 as one unsigned comparison per lane (max_epu32(t, 255) == 255)
        badi = _mm_or_si128(badi, _mm_xor_si128(_mm_max_epu32(ta, lim), lim));
        badi = _mm_or_si128(badi, _mm_xor_si128(_mm_max_epu32(tb, lim), lim));
        const __m128i w16 = _mm_packus_epi32(ta, tb);
        _mm_storel_epi64(reinterpret_cast<__m128i*>(dst + i), _mm_packus_epi16(w16, w16));
    }
    ok = _mm256_movemask_pd(bad) == 0 && _mm_testz_si128(badi, badi);
    return i;
}
#endif

static bool f64_to_u8(const double* src, size_t n, uint8_t* dst) {
    bool ok = true;
    size_t i0 = 0;
#if EF_X86
    if (has_avx2_bmi2()) i0 = f64_to_u8_avx2(src, n, dst, ok);
#endif
    for (size_t i = i0; i < n; ++i) {
        const double v = src[i];
        const bool in = v >= 0.0 && v <= 255.0;  // false for NaN
        const int t = in ? (int)v : 0;
        ok &= in && (double)t == v;
        dst[i] = (uint8_t)t;
    }
    return ok;
}

bool parallel_f64_to_u8(const double* src, size_t n, uint8_t* dst) {
    HostPool& P = host_pool();
    const size_t parts = std::min<size_t>((size_t)P.size(), std::max<size_t>(1, n >> 18));
    if (parts <= 1) return f64_to_u8(src, n, dst);
    const size_t per = (n / parts + 4095) & ~size_t(4095);
    Latch L;
    std::atomic<bool> all_ok{true};
    std::vector<std::pair<size_t, size_t>> ranges;
    for (size_t s = 0; s < n; s += per) ranges.emplace_back(s, std::min(n, s + per));
    L.add((int)ranges.size() - 1);
    for (size_t i = 1; i < ranges.size(); ++i) {
        const auto r = ranges[i];
        P.submit([=, &L, &all_ok] {
            if (!f64_to_u8(src + r.first, r.second - r.first, dst + r.first)) all_ok = false;
            L.done();
        }, true);
    }
    if (!f64_to_u8(src + ranges[0].first, ranges[0].second - ranges[0].first, dst + ranges[0].first)) all_ok = false;
    L.wait();
    return all_ok;
}

void parallel_copy(uint8_t* dst, const uint8_t* src, size_t bytes) {
    HostPool& P = host_pool();
    const size_t parts = std::min<size_t>((size_t)P.size(), std::max<size_t>(1, bytes >> 20));
    if (parts <= 1) {
        stream_copy(dst, src, bytes);
        return;
    }
    const size_t per = (bytes / parts + 4095) & ~size_t(4095);
    Latch L;
    size_t s = 0;
    std::vector<std::pair<size_t, size_t>> ranges;
    for (; s < bytes; s += per) ranges.emplace_back(s, std::min(bytes, s + per));
    L.add((int)ranges.size() - 1);
    for (size_t i = 1; i < ranges.size(); ++i) {
        const auto r = ranges[i];
        P.submit([=, &L] {
            stream_copy(dst + r.first, src + r.first, r.second - r.first);
            L.done();
        }, true);
    }
    stream_copy(dst + ranges[0].first, src + ranges[0].first, ranges[0].second - ranges[0].first);
    L.wait();
}

}  // namespace ef
