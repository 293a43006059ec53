// diffusion_tb.cuh — K1, temporally blocked (sm_100a).
//
// The 2048^2 diffusion field (2 slots x 16 MiB) is L2-resident, so the
// one-step kernel is bound by L2 latency and launch overhead, not HBM. Here a
// CTA pulls a (64 + 2HA)^2 patch of BOTH slots into shared memory with two
// TMA 2D box loads, advances it T <= TMAX steps in place (ping-pong; the
// valid region shrinks by R per step), and stores its 64^2 core of the last
// two levels: T steps per launch and 1/T of the global traffic. Every value
// is computed by exactly the single-step expression from the same neighbour
// values, so the result is bitwise the step-by-step run. Boundary cells
// (outside [R, n-R)) are never updated: each ping-pong buffer is loaded from
// the slot of matching level parity, so every level sees its own slot's
// boundary values (the reference's 2-slot loop), and the stored core carries
// those unchanged values back. Launches read one buffer pair and write the
// other, so tiles never race; the plan alternates pairs.
#pragma once

#include "tma_stencil.cuh"

namespace sfb {

struct DiffusionTBArgs {
    CUtensorMap src0;  // read pair, level parity 0: box (SW, SW)
    CUtensorMap src1;  // read pair, level parity 1
    float* dst[2];     // write pair, indexed by level parity
    int64_t pitch;
    int n0, n1;
    int t0;  // level at launch start
    int T;   // steps in this launch (<= TMAX)
    float c0;
    int has_c0;
    float cj[8];
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

template <int R>
__device__ __forceinline__ float diffusion_point(const DiffusionTBArgs& A, const float* c, int w) {
    float acc = 0.0f;
    bool first = true;
    if (A.has_c0) {
        acc = __fmul_rn(A.c0, c[0]);
        first = false;
    }
#pragma unroll
    for (int j = R; j >= 1; --j) {
        const float t = __fmul_rn(A.cj[j - 1], c[-j]);
        acc = first ? t : __fadd_rn(acc, t);
        first = false;
    }
#pragma unroll
    for (int j = 1; j <= R; ++j) acc = __fadd_rn(acc, __fmul_rn(A.cj[j - 1], c[j]));
#pragma unroll
    for (int j = R; j >= 1; --j) acc = __fadd_rn(acc, __fmul_rn(A.cj[j - 1], c[-j * w]));
#pragma unroll
    for (int j = 1; j <= R; ++j) acc = __fadd_rn(acc, __fmul_rn(A.cj[j - 1], c[j * w]));
    return acc;
}

// Four consecutive a1 cells of one row in the emitted order (centre if its
// weight is nonzero, a1 neighbours -R..-1, +1..+R, a0 neighbours -R..-1,
// +1..+R), from the row's aligned window and the a0 neighbour row vectors
// (up[j-1] = row -j, dn[j-1] = row +j).
template <int R, int RA>
__device__ __forceinline__ void diffusion_row4(const DiffusionTBArgs& A, const float* win,
                                               const float4* up, const float4* dn, float* acc) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float t = __fmul_rn(A.cj[R - 1], win[RA + k - R]);
        acc[k] = A.has_c0 ? __fadd_rn(__fmul_rn(A.c0, win[RA + k]), t) : t;
    }
#pragma unroll
    for (int j = R - 1; j >= 1; --j)
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] = __fadd_rn(acc[k], __fmul_rn(A.cj[j - 1], win[RA + k - j]));
#pragma unroll
    for (int j = 1; j <= R; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] = __fadd_rn(acc[k], __fmul_rn(A.cj[j - 1], win[RA + k + j]));
#pragma unroll
    for (int j = R; j >= 1; --j) {
        const float vv[4] = {up[j - 1].x, up[j - 1].y, up[j - 1].z, up[j - 1].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] = __fadd_rn(acc[k], __fmul_rn(A.cj[j - 1], vv[k]));
    }
#pragma unroll
    for (int j = 1; j <= R; ++j) {
        const float vv[4] = {dn[j - 1].x, dn[j - 1].y, dn[j - 1].z, dn[j - 1].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] = __fadd_rn(acc[k], __fmul_rn(A.cj[j - 1], vv[k]));
    }
}

template <int RA>
__device__ __forceinline__ void load_window(const float* c, float* win) {
#pragma unroll
    for (int q = 0; q < (4 + 2 * RA) / 4; ++q) {
        const float4 w = *reinterpret_cast<const float4*>(c - RA + 4 * q);
        win[4 * q] = w.x;
        win[4 * q + 1] = w.y;
        win[4 * q + 2] = w.z;
        win[4 * q + 3] = w.w;
    }
}

__device__ __forceinline__ void store_row4(float* o, int x, int ix0, int ix1, const float* acc) {
    if (x >= ix0 && x + 3 < ix1) {
        *reinterpret_cast<float4*>(o) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (x + k >= ix0 && x + k < ix1) o[k] = acc[k];
    }
}

// HA: load halo, TMAX*R rounded up to 4 (16-byte aligned box coordinates).
template <int R, int TILE, int TMAX>
struct TbLayout {
    static constexpr int HA = (TMAX * R + 3) / 4 * 4;
    static constexpr int SW = TILE + 2 * HA;
    static constexpr size_t smem = 128 + 2 * static_cast<size_t>(SW) * SW * sizeof(float);
};

// RV: rows per thread visit (1, or 2: two stacked rows share their a0
// neighbour loads -- each row's centre is the other's a0 neighbour -- and give
// each thread twice the independent work)
template <int R, int TILE, int TMAX, int RV = 1>
__global__ void __launch_bounds__(256) diffusion_tb_kernel(const __grid_constant__ DiffusionTBArgs A) {
    using L = TbLayout<R, TILE, TMAX>;
    constexpr int SW = L::SW, HA = L::HA;
    extern __shared__ __align__(128) unsigned char smraw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smraw);
    // buffer b at sbuf + b * SW * SW (pointer arithmetic on the shared
    // symbol keeps every access an LDS/STS; a pointer array would not)
    float* const sbuf = reinterpret_cast<float*>(smraw + 128);
    const int tid = threadIdx.x;
    const int tx = tid & 31, ty = tid >> 5;  // 32 x 8 (loads / stores)
    const int T = A.T;
    const int gx0 = blockIdx.x * TILE - HA;  // a1 of smem column 0
    const int gy0 = blockIdx.y * TILE - HA;  // a0 of smem row 0
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        mbar_arrive_expect_tx(bar, 2 * SW * SW * sizeof(float));
        // buffer b holds the slot of level parity (t0 + b)
        tma_load_2d(sbuf, (A.t0 & 1) ? &A.src1 : &A.src0, gx0, gy0, bar);
        tma_load_2d(sbuf + SW * SW, (A.t0 & 1) ? &A.src0 : &A.src1, gx0, gy0, bar);
    }
    mbar_wait(bar, 0);
    // (Packed fp32x2 arithmetic as in the acoustic kernels measured 3 %
    // slower here in the sustained C1 run, 747 vs 769 GPts/s: scalar. The
    // 64-wide core tile is the measured best for radius 1: 48 / 56 / 72 / 80
    // / 96 (SF_TB_TILE) ran at 699 / 714 / 677 / 654 / 599 vs 759 GPts/s;
    // two rows per visit (RV = 2) 776 vs 760.)
    // Each thread updates 4 consecutive a1 cells per visit: one aligned
    // (4 + 2RA)-float window (LDS.128s) gives every a1 neighbour, one
    // LDS.128 per a0 row offset gives the a0 neighbours of all four.
    constexpr int RA = (R + 3) / 4 * 4;
    // a pass covers whole smem rows: NV float4 columns x RPP rows (the
    // 66-78 wide valid region would leave most of a second 64-wide pass idle)
    constexpr int NV = SW / 4;
    constexpr int RPP = 256 / NV;
    const int lx = tid % NV, ly = tid / NV;
    for (int st = 1; st <= T; ++st) {
        const float* in = sbuf + ((st - 1) & 1) * (SW * SW);
        float* out = sbuf + (st & 1) * (SW * SW);
        // cells still valid after this step (core grown by (T - st) R)
        const int grow = HA - (T - st) * R;
        // global interior in smem coordinates
        const int iy0 = R - gy0, iy1 = A.n0 - R - gy0;
        const int ix0 = R - gx0, ix1 = A.n1 - R - gx0;
        const int ylo = max(grow, iy0), yhi = min(SW - grow, iy1);
        const int xlo = max(grow, ix0) & ~3, xhi = min(SW - grow, ix1);
        const int x = 4 * lx;
        const bool col_on = ly < RPP && x + 3 >= xlo && x < xhi;
        if (RV == 2) {
            for (int y = ylo + 2 * ly; col_on && y < yhi; y += 2 * RPP) {
                const bool two = y + 1 < yhi;
                const float* c0p = in + y * SW + x;
                const float* c1p = c0p + SW;
                float win0[4 + 2 * RA], win1[4 + 2 * RA];
                load_window<RA>(c0p, win0);
                float4 up0[R], dn0[R];
#pragma unroll
                for (int j = 1; j <= R; ++j) {
                    up0[j - 1] = *reinterpret_cast<const float4*>(c0p - j * SW);
                    dn0[j - 1] = *reinterpret_cast<const float4*>(c0p + j * SW);
                }
                float acc[4];
                diffusion_row4<R, RA>(A, win0, up0, dn0, acc);
                store_row4(out + y * SW + x, x, ix0, ix1, acc);
                if (two) {
                    // row y+1: its window's centre is dn0[0]; a0 neighbours are
                    // row y (win0's centre), up0 shifted by one, dn0 shifted
                    // by one and one more row below
#pragma unroll
                    for (int q = 0; q < (4 + 2 * RA) / 4; ++q) {  // centre chunk = dn0[0]
                        const float4 w = q == RA / 4 ? dn0[0]
                                                     : *reinterpret_cast<const float4*>(c1p - RA + 4 * q);
                        win1[4 * q] = w.x;
                        win1[4 * q + 1] = w.y;
                        win1[4 * q + 2] = w.z;
                        win1[4 * q + 3] = w.w;
                    }
                    float4 up1[R], dn1[R];
                    up1[0] = make_float4(win0[RA], win0[RA + 1], win0[RA + 2], win0[RA + 3]);
#pragma unroll
                    for (int j = 2; j <= R; ++j) up1[j - 1] = up0[j - 2];
#pragma unroll
                    for (int j = 1; j < R; ++j) dn1[j - 1] = dn0[j];
                    dn1[R - 1] = *reinterpret_cast<const float4*>(c1p + R * SW);
                    diffusion_row4<R, RA>(A, win1, up1, dn1, acc);
                    store_row4(out + (y + 1) * SW + x, x, ix0, ix1, acc);
                }
            }
        }
        for (int y = ylo + ly; RV == 1 && col_on && y < yhi; y += RPP) {
            {
                const float* c = in + y * SW + x;
                float win[4 + 2 * RA];
#pragma unroll
                for (int q = 0; q < (4 + 2 * RA) / 4; ++q) {
                    const float4 w = *reinterpret_cast<const float4*>(c - RA + 4 * q);
                    win[4 * q] = w.x;
                    win[4 * q + 1] = w.y;
                    win[4 * q + 2] = w.z;
                    win[4 * q + 3] = w.w;
                }
                float acc[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    // first emitted term: the centre when its weight is
                    // nonzero, else the a1 neighbour at offset -R
                    const float t = __fmul_rn(A.cj[R - 1], win[RA + k - R]);
                    acc[k] = A.has_c0 ? __fadd_rn(__fmul_rn(A.c0, win[RA + k]), t) : t;
                }
#pragma unroll
                for (int j = R - 1; j >= 1; --j)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        acc[k] = __fadd_rn(acc[k], __fmul_rn(A.cj[j - 1], win[RA + k - j]));
#pragma unroll
                for (int j = 1; j <= R; ++j)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        acc[k] = __fadd_rn(acc[k], __fmul_rn(A.cj[j - 1], win[RA + k + j]));
#pragma unroll
                for (int j = R; j >= 1; --j) {
                    const float4 v = *reinterpret_cast<const float4*>(c - j * SW);
                    const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        acc[k] = __fadd_rn(acc[k], __fmul_rn(A.cj[j - 1], vv[k]));
                }
#pragma unroll
                for (int j = 1; j <= R; ++j) {
                    const float4 v = *reinterpret_cast<const float4*>(c + j * SW);
                    const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        acc[k] = __fadd_rn(acc[k], __fmul_rn(A.cj[j - 1], vv[k]));
                }
                // cells outside the global interior keep their slot values;
                // cells outside the valid region may take any value (never read
                // by a valid cell), so only the interior test masks stores
                float* o = out + y * SW + x;
                if (x >= ix0 && x + 3 < ix1) {
                    *reinterpret_cast<float4*>(o) = make_float4(acc[0], acc[1], acc[2], acc[3]);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (x + k >= ix0 && x + k < ix1) o[k] = acc[k];
                }
            }
        }
        __syncthreads();
    }
    // core of the last two levels (boundary cells carry their slot's values)
#pragma unroll
    for (int lv = 0; lv < 2; ++lv) {
        const int level = A.t0 + T - lv;
        const float* b = sbuf + ((T - lv) & 1) * (SW * SW);
        float* d = A.dst[level & 1];
        for (int y = HA + ty; y < HA + TILE; y += 8) {
            const int gy = gy0 + y;
            if (gy >= A.n0) break;
            for (int x = HA + tx; x < HA + TILE; x += 32) {
                const int gx = gx0 + x;
                if (gx < A.n1) d[static_cast<int64_t>(gy) * A.pitch + gx] = b[y * SW + x];
            }
        }
    }
}

} // namespace sfb
