// ef_host.h -- host transfer helpers for ef_canny_u8_host (see ef_host.cu).
#pragma once
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <mutex>

#include <cuda_runtime.h>

namespace ef {

// 2-bit (labels, final) codes: 0 = (0, F), 1 = (1, F), 2 = (1, T), 3 = (2, T)
cudaError_t launch_pack(const uint8_t* labels, const uint8_t* final_map, long long n, uint8_t* packed, int sm_count,
                        cudaStream_t st);

// expand packed bytes [byte0, byte1) of an npx-pixel stream into labels/final_map
// (pointers address pixel 0 of the stream)
void unpack_codes(const uint8_t* packed, size_t byte0, size_t byte1, size_t npx, uint8_t* labels,
                  uint8_t* final_map);

// edges-only calls: the final map alone at 1 bit per pixel (bit k of byte j = pixel 8 j + k)
cudaError_t launch_pack_final(const uint8_t* final_map, long long n, uint8_t* packed, int sm_count, cudaStream_t st);
void unpack_bits(const uint8_t* packed, size_t byte0, size_t byte1, size_t npx, uint8_t* final_map);

void flush_lines(const uint8_t* p, size_t n);

class HostPool {
   public:
    explicit HostPool(int n);
    int size() const;
    void submit(std::function<void()> f, bool front = false);

   private:
    struct Impl;
    Impl* impl_;
};

HostPool& host_pool();

struct Latch {
    std::mutex mu;
    std::condition_variable cv;
    int count = 0;
    void add(int n);
    void done();
    void wait();
};

// memcpy split over the pool (used to stage pageable inputs into pinned memory)
void parallel_copy(uint8_t* dst, const uint8_t* src, size_t bytes);

// float64 -> u8 over the pool; true when every value is an integer in [0, 255]
bool parallel_f64_to_u8(const double* src, size_t n, uint8_t* dst);

}  // namespace ef
