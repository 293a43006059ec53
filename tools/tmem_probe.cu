// tools/tmem_probe.cu — TMEM as a per-thread register-file extension: latency
// and throughput of tcgen05.ld / tcgen05.st (32x32b shape: each lane its own
// row of 32-bit columns) on this B200. Sizing probe for a queue-vector
// stencil whose a0 register queue would live in TMEM.
//
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/tmem_probe tools/tmem_probe.cu
//   tools/tmem_probe          -> one JSON line per measurement
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    std::printf("{\"error\": \"%s at %d\"}\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int COLS>
__device__ __forceinline__ uint32_t tmem_alloc(uint32_t* slot) {
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(static_cast<uint32_t>(__cvta_generic_to_shared(slot))), "n"(COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    return *slot;
}

template <int COLS>
__device__ __forceinline__ void tmem_free(uint32_t base) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if ((threadIdx.x >> 5) == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(base), "n"(COLS));
}

// MODE 0: dependent load chain (latency): each load's column depends on the
// previous result. MODE 1: independent x16 loads, one wait per 4 (throughput).
// MODE 2: x4 stores + wait (write throughput).
template <int COLS, int MODE>
__global__ void __launch_bounds__(128) probe(int iters, unsigned long long* cycles, uint32_t* sink) {
    __shared__ uint32_t slot;
    const uint32_t base = tmem_alloc<COLS>(&slot);
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t taddr = base + ((32u * (warp & 3u)) << 16);
    uint32_t acc = threadIdx.x;
    // initialise the CTA's columns
    for (int c = 0; c < COLS; c += 4) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};"
                     :: "r"(taddr + c), "r"(acc), "r"(acc + 1), "r"(acc + 2), "r"(acc + 3));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    __syncthreads();
    const unsigned long long t0 = clock64();
    if (MODE == 0) {
        uint32_t col = 0;
        for (int i = 0; i < iters; ++i) {
            uint32_t v;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr + col));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            col = (v ^ col) & (COLS - 1) & ~0u;  // data-dependent address
            col &= 0;                            // keep it in range, still dependent
            acc += v;
        }
    } else if (MODE == 1) {
        for (int i = 0; i < iters; ++i) {
            uint32_t r[64];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t a = taddr + ((16 * (4 * i + k)) & (COLS - 1));
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                    : "=r"(r[16 * k + 0]), "=r"(r[16 * k + 1]), "=r"(r[16 * k + 2]), "=r"(r[16 * k + 3]),
                      "=r"(r[16 * k + 4]), "=r"(r[16 * k + 5]), "=r"(r[16 * k + 6]), "=r"(r[16 * k + 7]),
                      "=r"(r[16 * k + 8]), "=r"(r[16 * k + 9]), "=r"(r[16 * k + 10]), "=r"(r[16 * k + 11]),
                      "=r"(r[16 * k + 12]), "=r"(r[16 * k + 13]), "=r"(r[16 * k + 14]), "=r"(r[16 * k + 15])
                    : "r"(a));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 64; ++k) acc ^= r[k];
        }
    } else {
        for (int i = 0; i < iters; ++i) {
            const uint32_t a = taddr + ((4 * i) & (COLS - 1));
            asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};"
                         :: "r"(a), "r"(acc), "r"(acc + i), "r"(acc ^ i), "r"(acc + 7));
            if ((i & 3) == 3) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            acc += 3;
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    tmem_free<COLS>(base);
}

template <int COLS, int MODE>
int run(const char* name, int blocks, int iters, double bytes_per_iter_thread) {
    unsigned long long* cyc;
    uint32_t* sink;
    CK(cudaMalloc(&cyc, blocks * sizeof(unsigned long long)));
    CK(cudaMalloc(&sink, blocks * 128 * sizeof(uint32_t)));
    probe<COLS, MODE><<<blocks, 128>>>(iters, cyc, sink);  // warm
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    probe<COLS, MODE><<<blocks, 128>>>(iters, cyc, sink);
    cudaEventRecord(b);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[4096];
    CK(cudaMemcpy(h, cyc, blocks * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    double avg = 0;
    for (int i = 0; i < blocks; ++i) avg += static_cast<double>(h[i]);
    avg /= blocks;
    const double bytes = bytes_per_iter_thread * 128.0 * iters * blocks;
    std::printf("{\"probe\": \"%s\", \"cols\": %d, \"blocks\": %d, \"iters\": %d, \"cycles_per_iter\": %.2f, "
                "\"bytes_per_cycle_per_cta\": %.1f, \"chip_TBps\": %.2f, \"ms\": %.3f}\n",
                name, COLS, blocks, iters, avg / iters, bytes_per_iter_thread * 128.0 * iters / avg,
                bytes / (ms * 1e-3) / 1e12, ms);
    cudaFree(cyc);
    cudaFree(sink);
    return 0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<32, 0>("ld_x1_dependent_latency", 1, 4096, 4.0);
    run<128, 1>("ld_x16x4_throughput_1cta_per_sm", sms, 4096, 256.0);
    run<128, 1>("ld_x16x4_throughput_4cta_per_sm", 4 * sms, 4096, 256.0);
    run<128, 2>("st_x4_throughput_4cta_per_sm", 4 * sms, 16384, 16.0);
    return 0;
}
