// cluster_probe.cu — B200 measurements that size a two-step (t+1, t+2)
// stencil built on thread-block clusters: the cost of one
// cluster-wide barrier (arrive.release / wait.acquire) per plane, and the
// latency / bandwidth of distributed-shared-memory reads of a neighbour
// CTA's tile (ld.shared::cluster) against local LDS.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_probe cluster_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ void cluster_sync_rel_acq() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ITERS cluster barriers back to back; clock64 per CTA
__global__ void barrier_kernel(int iters, long long* cycles) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) cluster_sync_rel_acq();
    long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// dependent-chain latency of loads from the neighbour CTA's shared memory
// (remote = 1) or the own CTA's (remote = 0)
__global__ void dsmem_latency_kernel(int iters, int remote, long long* cycles, int* sink) {
    __shared__ int buf[1024];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i * 37 + 11) & 1023;
    cl.sync();
    const unsigned rank = cl.block_rank();
    int* src = remote ? cl.map_shared_rank(buf, (rank + 1) % cl.num_blocks()) : buf;
    int idx = threadIdx.x & 1023;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) idx = src[idx];
    long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = idx;
    cl.sync();
}

// streaming 16-byte reads of a neighbour's (or the own) 32 KB tile
__global__ void dsmem_bw_kernel(int iters, int remote, float* sink) {
    __shared__ float4 buf[2048];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_float4(i, i, i, i);
    cl.sync();
    const unsigned rank = cl.block_rank();
    float4* src = remote ? cl.map_shared_rank(buf, (rank + 1) % cl.num_blocks()) : buf;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int it = 0; it < iters; ++it)
        for (int i = threadIdx.x; i < 2048; i += blockDim.x) {
            const float4 v = src[(i + it) & 2047];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
    cl.sync();
}

template <typename K, typename... Args>
float launch_cluster(K kernel, int csize, int blocks, int threads, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args...);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = -1;
    if (e == cudaSuccess) cudaEventElapsedTime(&ms, a, b);
    else printf("{\"error\":\"%s\"}\n", cudaGetErrorString(e));
    return ms;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* cyc;
    int* isink;
    float* fsink;
    const int maxb = sms * 8;
    cudaMalloc(&cyc, sizeof(long long) * maxb);
    cudaMalloc(&isink, sizeof(int) * maxb * 256);
    cudaMalloc(&fsink, sizeof(float) * maxb * 256);
    long long h[2048];
    for (int cs : {2, 4, 8}) {
        const int blocks = (sms / cs) * cs;
        const int iters = 10000;
        launch_cluster(barrier_kernel, cs, blocks, 256, iters, cyc);
        launch_cluster(barrier_kernel, cs, blocks, 256, iters, cyc);
        cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
        double s = 0;
        for (int i = 0; i < blocks; ++i) s += h[i];
        printf("{\"probe\":\"cluster_barrier\",\"cluster\":%d,\"threads\":256,\"cycles_per_barrier\":%.1f}\n",
               cs, s / blocks / iters);
        for (int remote = 0; remote < 2; ++remote) {
            const int li = 4096;
            launch_cluster(dsmem_latency_kernel, cs, blocks, 32, li, remote, cyc, isink);
            cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
            double t = 0;
            for (int i = 0; i < blocks; ++i) t += h[i];
            printf("{\"probe\":\"smem_load_latency\",\"cluster\":%d,\"remote\":%d,\"cycles\":%.1f}\n", cs,
                   remote, t / blocks / li);
            const int bi = 2000;
            launch_cluster(dsmem_bw_kernel, cs, sms * 2 / cs * cs, 512, 10, remote, fsink);
            const float ms = launch_cluster(dsmem_bw_kernel, cs, sms * 2 / cs * cs, 512, bi, remote, fsink);
            const double bytes = double(sms * 2 / cs * cs) * 2048.0 * 16.0 * bi;
            printf("{\"probe\":\"smem_read_bw\",\"cluster\":%d,\"remote\":%d,\"GBps_total\":%.0f}\n", cs, remote,
                   bytes / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
