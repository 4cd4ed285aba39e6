// Host-side probe: pinned PCIe bandwidth (H2D, D2H, both) and 2-bit unpack throughput.
#include <cuda_runtime.h>
#include <immintrin.h>
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

static uint32_t LUT_L[256], LUT_F[256];
static void unpack(const uint8_t* p, size_t nbytes, uint8_t* lab, uint8_t* fin, bool nt) {
    size_t i = 0;
    if (nt) {
        for (; i + 4 <= nbytes; i += 4) {
            __m128i l = _mm_setr_epi32(LUT_L[p[i]], LUT_L[p[i + 1]], LUT_L[p[i + 2]], LUT_L[p[i + 3]]);
            __m128i f = _mm_setr_epi32(LUT_F[p[i]], LUT_F[p[i + 1]], LUT_F[p[i + 2]], LUT_F[p[i + 3]]);
            _mm_stream_si128((__m128i*)(lab + 4 * i), l);
            _mm_stream_si128((__m128i*)(fin + 4 * i), f);
        }
        _mm_sfence();
    }
    for (; i < nbytes; ++i) { memcpy(lab + 4 * i, &LUT_L[p[i]], 4); memcpy(fin + 4 * i, &LUT_F[p[i]], 4); }
}
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
    for (int b = 0; b < 256; ++b) {
        uint32_t l = 0, f = 0;
        for (int k = 0; k < 4; ++k) {
            int c = (b >> (2 * k)) & 3;
            l |= (uint32_t)(c == 0 ? 0 : c == 3 ? 2 : 1) << (8 * k);
            f |= (uint32_t)(c >= 2) << (8 * k);
        }
        LUT_L[b] = l; LUT_F[b] = f;
    }
    const size_t N = 132710400;
    uint8_t *hs, *hl, *hf, *d1, *d2;
    cudaMallocHost(&hs, N); cudaMallocHost(&hl, 2 * N); hf = hl + N;
    cudaMalloc(&d1, N); cudaMalloc(&d2, 2 * N);
    memset(hs, 1, N); memset(hl, 0, 2 * N);
    cudaStream_t a, b; cudaStreamCreate(&a); cudaStreamCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        double t = now(); cudaMemcpyAsync(d1, hs, N, cudaMemcpyHostToDevice, a); cudaStreamSynchronize(a);
        double h2d = N / (now() - t) / 1e9;
        t = now(); cudaMemcpyAsync(hl, d2, 2 * N, cudaMemcpyDeviceToHost, a); cudaStreamSynchronize(a);
        double d2h = 2 * N / (now() - t) / 1e9;
        t = now(); cudaMemcpyAsync(d1, hs, N, cudaMemcpyHostToDevice, a); cudaMemcpyAsync(hl, d2, 2 * N, cudaMemcpyDeviceToHost, b);
        cudaDeviceSynchronize(); double both = now() - t;
        printf("pinned H2D %.1f GB/s  D2H %.1f GB/s  both(1+2 B/px) %.2f ms\n", h2d, d2h, both * 1e3);
    }
    // pageable destination D2H
    std::vector<uint8_t> pg(2 * N, 0);
    { double t = now(); cudaMemcpy(pg.data(), d2, 2 * N, cudaMemcpyDeviceToHost); printf("pageable D2H %.1f GB/s\n", 2 * N / (now() - t) / 1e9); }
    std::vector<uint8_t> packed(N / 4);
    for (size_t i = 0; i < packed.size(); ++i) packed[i] = (uint8_t)(i * 37 + (i >> 9));
    for (int nt = 0; nt < 2; ++nt)
        for (int T : {1, 4, 8, 12, 16}) {
            for (int rep = 0; rep < 2; ++rep) {
                double t = now();
                std::vector<std::thread> th;
                size_t per = (packed.size() / T + 63) & ~size_t(63);
                for (int k = 0; k < T; ++k) {
                    size_t s = std::min(packed.size(), k * per), e = std::min(packed.size(), s + per);
                    th.emplace_back([&, s, e] { unpack(packed.data() + s, e - s, hl + 4 * s, hf + 4 * s, nt); });
                }
                for (auto& x : th) x.join();
                double dt = now() - t;
                if (rep) printf("unpack nt=%d T=%2d: %.2f ms (%.1f GB/s written)\n", nt, T, dt * 1e3, 2 * N / dt / 1e9);
            }
        }
    // concurrency: H2D stream of the whole input while T threads unpack
    for (int T : {2, 4, 8, 12, 16}) {
        std::vector<std::thread> th;
        double t0 = now();
        for (int k = 0; k < T; ++k) {
            size_t per = (packed.size() / T + 63) & ~size_t(63);
            size_t s = std::min(packed.size(), k * per), e = std::min(packed.size(), s + per);
            th.emplace_back([&, s, e] { unpack(packed.data() + s, e - s, hl + 4 * s, hf + 4 * s, true); });
        }
        double t1 = now();
        cudaMemcpyAsync(d1, hs, N, cudaMemcpyHostToDevice, a); cudaStreamSynchronize(a);
        double h2d_t = now() - t1;
        for (auto& x : th) x.join();
        double all_t = now() - t0;
        printf("concurrent T=%2d: H2D %.1f GB/s (%.2f ms), unpack+H2D total %.2f ms\n", T, N / h2d_t / 1e9, h2d_t * 1e3, all_t * 1e3);
    }
    // unpack into pageable (first-touch vs warm)
    {
        std::vector<uint8_t> L(N), F(N);
        for (int rep = 0; rep < 2; ++rep) {
            double t = now();
            std::vector<std::thread> th;
            int T = 16; size_t per = (packed.size() / T + 63) & ~size_t(63);
            for (int k = 0; k < T; ++k) {
                size_t s = std::min(packed.size(), k * per), e = std::min(packed.size(), s + per);
                th.emplace_back([&, s, e] { unpack(packed.data() + s, e - s, L.data() + 4 * s, F.data() + 4 * s, true); });
            }
            for (auto& x : th) x.join();
            printf("unpack pageable T=16 rep %d: %.2f ms\n", rep, (now() - t) * 1e3);
        }
    }
    return 0;
}
