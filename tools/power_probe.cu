// power_probe.cu — what the 1 kW board power cap leaves for exact fp32 work and
// HBM streaming on one B200: runs, for a few seconds each, (a) a register-only
// FMUL2 / FFMA2(x, ONE, y) loop (the stencils' arithmetic form, pk2.cuh), (b)
// a float4 copy stream over buffers far larger than L2, (c) both at once on
// two streams with the fp kernel limited to a share of the SMs' issue time,
// and prints the sustained rates. tools/power_probe.py samples nvidia-smi
// power / SM clock next to it.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o power_probe power_probe.cu
//   ./power_probe <mode: fp|copy|both> <seconds> [fp_duty_percent]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

typedef unsigned long long u64;

__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
    u64 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 add2o(u64 a, u64 b, u64 one) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(one), "l"(b));
    return r;
}

constexpr int CH = 8;

// acc = acc + k * x per chain: one FMUL2 and one FFMA2 (4 fp32 operations)
// per chain-iteration; `sleep_ns` > 0 idles the warp between bursts to set a
// duty cycle
__global__ void fp_kernel(float* out, u64 k, u64 one, int iters, int bursts, unsigned sleep_ns) {
    u64 acc[CH], x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        acc[c] = k + threadIdx.x + c;
        x[c] = k ^ (static_cast<u64>(c) << 20);
    }
    for (int b = 0; b < bursts; ++b) {
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                acc[c] = add2o(acc[c], mul2(k, x[c]), one);
                x[c] = acc[c];  // keeps the FMUL2 inside the loop (no extra instruction)
            }
        }
        if (sleep_ns) __nanosleep(sleep_ns);
    }
    u64 s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s ^= acc[c];
    if (s == 0x1234567ull) out[0] = 1.0f;
}

// shared-memory read stream: LDS.128 per lane from conflict-free addresses,
// results folded with one XOR per load so they are not dead
__global__ void lds_kernel(float* out, int iters) {
    __shared__ uint4 buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_uint4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    uint4 s = make_uint4(0, 0, 0, 0);
    int idx = threadIdx.x;
    const unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(buf));
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            uint4 v;  // volatile: the loads stay in the loop
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "r"(base + 16u * ((idx + 32 * u) & 1023)));
            s.x ^= v.x;
            s.y ^= v.y;
            s.z ^= v.z;
            s.w ^= v.w;
        }
        idx += 256;
    }
    if ((s.x ^ s.y ^ s.z ^ s.w) == 0x12345u) out[0] = 1.0f;
}

// register moves on the ALU pipe (PRMT identity), 16 independent registers
__global__ void mov_kernel(float* out, int iters) {
    unsigned r[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) r[c] = threadIdx.x + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 16; ++c) asm volatile("prmt.b32 %0, %1, 0, 0x3210;" : "=r"(r[c]) : "r"(r[(c + 1) & 15]));
    }
    unsigned s = 0;
#pragma unroll
    for (int c = 0; c < 16; ++c) s ^= r[c];
    if (s == 0x12345u) out[0] = 1.0f;
}

__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
    size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (; i < n; i += stride) b[i] = a[i];
}

int main(int argc, char** argv) {
    const char* mode = argc > 1 ? argv[1] : "fp";
    const double seconds = argc > 2 ? atof(argv[2]) : 5.0;
    const int duty = argc > 3 ? atoi(argv[3]) : 100;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    if (!strcmp(mode, "lds") || !strcmp(mode, "mov") || !strcmp(mode, "l2")) {
        float* o;
        cudaMalloc(&o, 4096);
        cudaEvent_t a0, a1;
        cudaEventCreate(&a0);
        cudaEventCreate(&a1);
        const size_t l2n = (48ull << 20) / 16;  // 48 MiB source + 48 MiB destination: L2-resident
        float4 *la = nullptr, *lb = nullptr;
        if (!strcmp(mode, "l2")) {
            cudaMalloc(&la, l2n * 16);
            cudaMalloc(&lb, l2n * 16);
            cudaMemset(la, 1, l2n * 16);
        }
        double units = 0;
        const auto t0 = std::chrono::steady_clock::now();
        cudaEventRecord(a0);
        while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < seconds) {
            for (int r = 0; r < 8; ++r) {
                if (!strcmp(mode, "lds")) {
                    lds_kernel<<<4 * nsm, 256>>>(o, 4096);
                    units += 4.0 * nsm * 256 * 4096.0 * 8 * 16;  // bytes read from shared memory
                } else if (!strcmp(mode, "mov")) {
                    mov_kernel<<<4 * nsm, 256>>>(o, 4096);
                    units += 4.0 * nsm * 256 * 4096.0 * 16;  // thread-instructions
                } else {
                    copy_kernel<<<nsm * 8, 512>>>(la, lb, l2n);
                    units += 2.0 * l2n * 16;  // bytes through L2
                }
            }
            cudaDeviceSynchronize();
        }
        cudaEventRecord(a1);
        cudaEventSynchronize(a1);
        float ms = 0;
        cudaEventElapsedTime(&ms, a0, a1);
        printf("{\"probe\":\"power\",\"mode\":\"%s\",\"seconds\":%.2f,\"%s\":%.2f}\n", mode, ms / 1e3,
               !strcmp(mode, "mov") ? "thread_tinstr_per_s" : !strcmp(mode, "lds") ? "smem_read_tbs" : "l2_tbs",
               units / ms / 1e9);
        return 0;
    }
    const bool do_fp = strcmp(mode, "copy") != 0, do_copy = strcmp(mode, "fp") != 0;
    cudaStream_t sf, sc;
    cudaStreamCreate(&sf);
    cudaStreamCreate(&sc);
    float* out;
    cudaMalloc(&out, 4096);
    const size_t n4 = (4ull << 30) / 16;  // 4 GiB per buffer
    float4 *a = nullptr, *b = nullptr;
    if (do_copy) {
        cudaMalloc(&a, n4 * 16);
        cudaMalloc(&b, n4 * 16);
        cudaMemset(a, 1, n4 * 16);
    }
    const float2 one2 = make_float2(1.0f, 1.0f), k2 = make_float2(1.23e-4f, -1.17e-4f);
    u64 one, k;
    memcpy(&one, &one2, 8);
    memcpy(&k, &k2, 8);
    // fp launch: 2 CTAs of 256 threads per SM (room left for the copy's CTAs)
    const int iters = 256, bursts = 64;
    // busy time of a burst ~ iters * CH * 2 instr * 2 cycles * (warps per SMSP = 4) / 1.8 GHz
    const double burst_ns = iters * CH * 2 * 2.0 * 4 / 1.8;
    const unsigned sleep_ns = duty >= 100 ? 0u : static_cast<unsigned>(burst_ns * (100 - duty) / duty);
    const double fp_ops_per_launch = 4.0 * CH * iters * bursts * 256.0 * (2.0 * nsm);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double fp_ops = 0, bytes = 0;
    const auto t0 = std::chrono::steady_clock::now();
    cudaEventRecord(e0);
    int rounds = 0;
    while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < seconds) {
        for (int r = 0; r < 4; ++r) {
            if (do_fp) {
                fp_kernel<<<2 * nsm, 256, 0, sf>>>(out, k, one, iters, bursts, sleep_ns);
                fp_ops += fp_ops_per_launch;
            }
            if (do_copy) {
                copy_kernel<<<nsm * 8, 512, 0, sc>>>(a, b, n4);
                bytes += 2.0 * n4 * 16;
            }
        }
        cudaStreamSynchronize(sf);
        cudaStreamSynchronize(sc);
        ++rounds;
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\":\"power\",\"mode\":\"%s\",\"duty\":%d,\"seconds\":%.2f,\"fp32_tops\":%.2f,"
           "\"hbm_gbs\":%.1f}\n",
           mode, duty, ms / 1e3, fp_ops / ms / 1e9, bytes / ms / 1e6);
    return 0;
}
