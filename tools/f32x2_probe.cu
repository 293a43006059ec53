// f32x2_probe.cu — measures issue/throughput of scalar FMUL/FADD against the
// packed FMUL2/FADD2/FFMA2 forms on one B200, and checks that the packed
// forms round exactly like the scalar ones (the stencil kernels must stay
// bitwise equal to the reference's -ffp-contract=off C).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o f32x2_probe f32x2_probe.cu
//
// Note on contraction: ptxas fuses `mul.rn.f32x2` feeding `add.rn.f32x2`
// into FFMA2 even with --fmad=false. The contraction-proof form used here
// (and in the stencil kernels) is: products as FMUL2, sums as
// fma.rn.f32x2(a, ONE, b) with ONE an opaque register (ptxas cannot prove it
// is 1.0, so cannot fold the product into it). a*1 + b rounds once, exactly
// like a + b.
#include <cstdio>
#include <cstdint>
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

constexpr int CH = 8;  // independent chains per thread

// acc = acc + k*x (scalar, unfused), ITER times per chain
__global__ void scalar_kernel(float* out, float k, int iters) {
    float acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { acc[c] = threadIdx.x * 1e-3f + c; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[c] = __fadd_rn(acc[c], __fmul_rn(k, acc[c]));
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// the same 2*CH fp32 ops per iteration, as CH/2 packed pairs (each pair = two
// scalar chains): FMUL2 + FFMA2(one)
__global__ void packed_kernel(float* out, float k, int iters, u64 one) {
    u64 acc[CH / 2], x[CH / 2];
    const float2 kk2 = make_float2(k, k);
    u64 kk;
    memcpy(&kk, &kk2, 8);
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) {
        float2 a = make_float2(threadIdx.x * 1e-3f + 2 * c, threadIdx.x * 1e-3f + 2 * c + 1);
        float2 b = make_float2(1.0f + 2 * c * 1e-4f, 1.0f + (2 * c + 1) * 1e-4f);
        memcpy(&acc[c], &a, 8);
        memcpy(&x[c], &b, 8);
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH / 2; ++c) acc[c] = add2o(acc[c], mul2(kk, acc[c]), one);
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) {
        float2 a;
        memcpy(&a, &acc[c], 8);
        s += a.x + a.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// bitwise check of the packed forms against scalar rn ops on random bit patterns
__global__ void check_kernel(const uint32_t* a, const uint32_t* b, const uint32_t* c, int n,
                             u64 one, unsigned long long* bad) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * i + 1 >= n) return;
    float a0 = __uint_as_float(a[2 * i]), a1 = __uint_as_float(a[2 * i + 1]);
    float b0 = __uint_as_float(b[2 * i]), b1 = __uint_as_float(b[2 * i + 1]);
    float c0 = __uint_as_float(c[2 * i]), c1 = __uint_as_float(c[2 * i + 1]);
    float s0 = __fadd_rn(c0, __fmul_rn(a0, b0)), s1 = __fadd_rn(c1, __fmul_rn(a1, b1));
    u64 A, B, C;
    float2 t;
    t = make_float2(a0, a1); memcpy(&A, &t, 8);
    t = make_float2(b0, b1); memcpy(&B, &t, 8);
    t = make_float2(c0, c1); memcpy(&C, &t, 8);
    u64 R = add2o(C, mul2(A, B), one);
    float2 r;
    memcpy(&r, &R, 8);
    auto same = [](float x, float y) {
        return __float_as_uint(x) == __float_as_uint(y) || (x != x && y != y);
    };
    if (!same(r.x, s0) || !same(r.y, s1)) atomicAdd(bad, 1ull);
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 256, blocks = nsm * 8, iters = 1 << 14;
    float* out;
    cudaMalloc(&out, sizeof(float) * threads * blocks);
    const float2 one2 = make_float2(1.0f, 1.0f);
    u64 one;
    memcpy(&one, &one2, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double ops = 2.0 * CH * iters * (double)threads * blocks;
    for (int rep = 0; rep < 3; ++rep) {
        float ms_s, ms_p;
        cudaEventRecord(e0);
        scalar_kernel<<<blocks, threads>>>(out, 1.000001f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms_s, e0, e1);
        cudaEventRecord(e0);
        packed_kernel<<<blocks, threads>>>(out, 1.000001f, iters, one);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms_p, e0, e1);
        printf("{\"probe\":\"fp32_throughput\",\"scalar_tops\":%.2f,\"packed_tops\":%.2f,"
               "\"scalar_ms\":%.3f,\"packed_ms\":%.3f}\n",
               ops / ms_s / 1e9, ops / ms_p / 1e9, ms_s, ms_p);
    }
    // bitwise check on 64M random bit patterns (including NaN/inf/denormals)
    const int n = 1 << 26;
    uint32_t *a, *b, *c;
    cudaMallocManaged(&a, 4ull * n);
    cudaMallocManaged(&b, 4ull * n);
    cudaMallocManaged(&c, 4ull * n);
    uint64_t s = 0x9E3779B97F4A7C15ull;
    auto nxt = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (uint32_t)s; };
    for (int i = 0; i < n; ++i) {
        a[i] = nxt();
        b[i] = nxt();
        c[i] = nxt();
        if ((i & 7) == 1) b[i] = (a[i] & 0x807fffffu) | ((254u - ((a[i] >> 23) & 0xff)) << 23);
        if ((i & 7) == 2) c[i] = a[i] ^ 0x80000000u;
    }
    unsigned long long* bad;
    cudaMallocManaged(&bad, 8);
    *bad = 0;
    check_kernel<<<(n / 2 + 255) / 256, 256>>>(a, b, c, n, one, bad);
    cudaError_t err = cudaDeviceSynchronize();
    printf("{\"probe\":\"packed_bitwise\",\"pairs\":%d,\"mismatches\":%llu,\"err\":\"%s\"}\n", n / 2,
           *bad, cudaGetErrorString(err));
    return 0;
}
