// pipe_probe.cu — per-SM throughput of the fp32 instruction forms the stencil
// kernels can use (scalar FMUL/FADD/FFMA, packed FMUL2/FFMA2, the
// contraction-proof a*ONE+b sum, IMAD), in SASS warp-instructions per SM
// clock, from %clock64 around fully resident grids.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o pipe_probe pipe_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

typedef unsigned long long u64;

constexpr int CH = 8;      // independent chains per thread
constexpr int ITERS = 2048;

__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
    u64 r;
    asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
    u64 r;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
    u64 r;
    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ float fmul(float a, float b) {
    float r;
    asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float fadd(float a, float b) {
    float r;
    asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float ffma(float a, float b, float c) {
    float r;
    asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

struct Rec {
    long long t0, t1;
    int smid;
};

__device__ __forceinline__ int smid() {
    int s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    return s;
}

// MODE: 0 FMUL r,r   1 FADD r,r   2 FFMA r,r,r   3 FMUL2 r,r   4 FFMA2 r,r,r
//       5 FFMA2 r,ONE(param),r   6 FADD2 r,r   7 IMAD r,r,r   8 FMUL r,const
//       9 mac pair: FMUL2 r,r + FFMA2 r,ONE,r (the stencil's term)
//      10 mul.rn.f32x2 feeding add.rn.f32x2 (does ptxas contract it?)
template <int MODE>
__global__ void probe(float* out, Rec* rec, float k, u64 one, int iters) {
    __shared__ long long t0s;
    const int tid = threadIdx.x;
    float a[CH], b[CH];
    u64 p[CH], q[CH];
    unsigned ia[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        a[c] = tid * 1e-3f + c;
        b[c] = 1.0f + c * 1e-5f + tid * 1e-9f + k * 1e-7f;
        float2 x = make_float2(a[c], a[c] + 0.5f), y = make_float2(b[c], b[c] + 1e-6f * tid);
        memcpy(&p[c], &x, 8);
        memcpy(&q[c], &y, 8);
        ia[c] = tid + c;
    }
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (MODE == 0) a[c] = fmul(a[c], b[c]);
            if (MODE == 1) a[c] = fadd(a[c], b[c]);
            if (MODE == 2) a[c] = ffma(a[c], b[c], a[c]);
            if (MODE == 3) p[c] = mul2(p[c], q[c]);
            if (MODE == 4) p[c] = fma2(p[c], q[c], p[c]);
            if (MODE == 5) p[c] = fma2(p[c], one, q[c]);
            if (MODE == 6) p[c] = add2(p[c], q[c]);
            if (MODE == 7) ia[c] = ia[c] * ia[(c + 1) % CH] + ia[c];
            if (MODE == 8) a[c] = fmul(a[c], k);
            if (MODE == 9) p[c] = fma2(mul2(q[(c + 3) % CH], p[(c + 1) % CH]), one, p[c]);
            if (MODE == 10) p[c] = add2(mul2(q[(c + 3) % CH], p[(c + 1) % CH]), p[c]);
        }
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        float2 x;
        memcpy(&x, &p[c], 8);
        s += a[c] + x.x + x.y + (float)ia[c];
    }
    out[blockIdx.x * blockDim.x + tid] = s;
    if (tid == 0) {
        t0s = t0;
    }
    __syncthreads();
    if (tid == 0) rec[blockIdx.x] = {t0s, t1, smid()};
}

template <int MODE>
void run(const char* name, int instr_per_chain_iter, int nsm) {
    const int threads = 256, blocks = nsm * 8;
    float* out;
    Rec* rec;
    cudaMalloc(&out, sizeof(float) * threads * blocks);
    cudaMalloc(&rec, sizeof(Rec) * blocks);
    float2 o = make_float2(1.0f, 1.0f);
    u64 one;
    memcpy(&one, &o, 8);
    probe<MODE><<<blocks, threads>>>(out, rec, 1.0001f, one, ITERS);  // warm
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<MODE><<<blocks, threads>>>(out, rec, 1.0001f, one, ITERS);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    Rec* h = new Rec[blocks];
    cudaMemcpy(h, rec, sizeof(Rec) * blocks, cudaMemcpyDeviceToHost);
    // per SM: warp-instructions of all its blocks / (max t1 - min t0)
    double sum_rate = 0;
    int nrate = 0;
    for (int s = 0; s < nsm; ++s) {
        long long lo = -1, hi = 0;
        int nb = 0;
        for (int b = 0; b < blocks; ++b)
            if (h[b].smid == s) {
                lo = lo < 0 || h[b].t0 < lo ? h[b].t0 : lo;
                hi = h[b].t1 > hi ? h[b].t1 : hi;
                ++nb;
            }
        if (nb == 0) continue;
        double winstr = double(nb) * (threads / 32) * ITERS * CH * instr_per_chain_iter;
        sum_rate += winstr / double(hi - lo);
        ++nrate;
    }
    const double lane_ops = double(blocks) * threads * ITERS * CH * instr_per_chain_iter;
    printf("{\"probe\": \"%s\", \"warp_instr_per_clk_per_sm\": %.3f, \"thread_instr_per_s\": %.4g, "
           "\"ms\": %.3f}\n",
           name, sum_rate / nrate, lane_ops / (ms * 1e-3), ms);
    delete[] h;
    cudaFree(out);
    cudaFree(rec);
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    run<0>("FMUL r,r", 1, nsm);
    run<8>("FMUL r,const", 1, nsm);
    run<1>("FADD r,r", 1, nsm);
    run<2>("FFMA r,r,r", 1, nsm);
    run<3>("FMUL2 r,r", 1, nsm);
    run<4>("FFMA2 r,r,r", 1, nsm);
    run<5>("FFMA2 r,ONE,r", 1, nsm);
    run<6>("FADD2 r,r (as compiled)", 1, nsm);
    run<7>("IMAD r,r,r", 1, nsm);
    run<9>("FMUL2+FFMA2(ONE) pair", 2, nsm);
    run<10>("mul.f32x2 + add.f32x2 pair (as compiled)", 2, nsm);
    return 0;
}
