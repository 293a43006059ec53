// tma_stencil.cuh — TMA/mbarrier-pipelined 3D acoustic stencil (sm_100a).
//
// Same arithmetic contract as kernels.cuh (the reference's emitted fp32
// expression, operation for operation). What changes is how data reaches
// the SM: instead of per-thread loads, one elected thread drives the Tensor
// Memory Accelerator, which streams 3D boxes of every input plane into a
// shared-memory pipeline S planes ahead of the compute:
//
//   cur ring  : 2R+S slots, each the (32*NX + 2RA) x (TY + 2R) box of u(t) at
//               one a0 plane, halo included (TMA zero-fills out-of-range
//               boxes at the grid faces, which only feed non-stored points);
//               the a0 neighbours of plane z are the same (a1, a2) position
//               in the slots of planes z-R..z+R, so no register queue;
//   pme stage : S slots of the (32*NX) x TY boxes of u(t-1), m, eta.
//
// Group i (iteration z = zb + i) = cur plane z+R + the u(t-1)/m/eta boxes of
// plane z, completing on mbarrier i % S (expect_tx = its byte count). After
// computing plane z every thread passes one __syncthreads; thread 0 then
// re-arms that barrier and issues group i+S into the slots just released
// (cur plane z-R, pme slot of z). Loads cost no registers and no LSU issue
// slots, so warps only spend issue bandwidth on the math and the LDS of the
// neighbours; the output is written with coalesced 128-byte stores.
#pragma once

#include <cuda.h>
#include <cstdint>

#include "kernels.cuh"
#include "pk2.cuh"

namespace sfb {

// All maps are 4D (a2, a1, a0, level): a time slot is a 1-level map, the
// FWI wavefield history an (nt+2)-level one; lv_* select the level.
struct TmaStencilArgs {
    CUtensorMap cur;   // box (WB, TY+2R, 1, 1) at (x0-RA, y0-R, z, lv_cur)
    CUtensorMap prev;  // box (TX, TY, 1, 1)
    CUtensorMap m;     // box (TX, TY, 1, 1)
    CUtensorMap eta;   // box (TX, TY, 1, 1)
    CUtensorMap old;   // GRAD: the output slot before it is overwritten (v(t+2))
    CUtensorMap uh;    // GRAD: forward history, level lv_uh = u(t+1)
    CUtensorMap grad;  // GRAD: gradient accumulator
    CUtensorMap cur_core;  // vecq2: un-halo'd box (TX, TY) of the cur level
    float* out;
    float* gradp;
    const float* cur_ptr;  // base of the cur map's field (vecq queue-head loads)
    int64_t level_elems;   // elements per level of the cur map
    int lv_cur, lv_prev, lv_uh;
    int pitch, plane;  // elements
    int n0, n1, n2;
    int zchunk;
    int z0, z1;  // planes of axis 0 this launch updates
    int stages;
    float ce, cm;
    float tc[3];
    float c0;
    float cj[8];
    // the same constants as (c, c) pairs for the packed fp32x2 kernels, and
    // the opaque ONE their sums multiply by (pk2.cuh)
    unsigned long long pk_one, pk_ce, pk_cm, pk_tc[3], pk_c0, pk_cj[8];
    // eta boxes known to be all +0.0 (the undamped interior): bit z of
    // eta0[(tile_y * eta0_ntx + tile_x) * eta0_words + z / 32]. The vector
    // kernels skip those boxes' TMA loads and use 0.0f, which is bitwise the
    // value they would have read (null = load every box).
    const uint32_t* eta0;
    int eta0_ntx, eta0_words;
    // Fused sparse epilogue (vector ring kernel): after its last plane a CTA
    // (1) injects this step's sources into the cells of its own tile (a
    // tile-sorted copy of the injection CSR: cells [tile_start[b],
    // tile_start[b+1]) belong to CTA b) and (2) samples the PREVIOUS step's
    // receivers from `cur`, which this step does not write. Null / 0 = off.
    const int* inj_tile_start;
    const int64_t* inj_cell;
    const int* inj_start;
    const int* inj_cp;
    const float* inj_cw;
    const float* inj_row;  // series row of this step
    const float* mfield;   // m (the injection divides by it)
    float inj_scale;
    const float* smp_field;
    const int* smp_ci;
    const float* smp_w;
    float* smp_out;        // series row of the previous step
    int smp_np;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// Bounded wait: a transaction count that never completes (a box/byte-count
// mismatch) traps after ~2^24 suspended polls instead of hanging the GPU.
// Wait for a phase of an mbarrier. try_wait with a suspend-time hint lets the
// hardware park the warp until the phase completes (or the hint expires)
// instead of re-issuing the poll: spinning waiters otherwise take issue slots
// from the compute warps of the same scheduler. Bounded: a wait that never
// completes (a TMA fault, a mis-sized box) traps instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait_addr(uint32_t addr, uint32_t parity) {
    uint32_t done = 0;
    for (uint32_t spins = 0;; ++spins) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(addr), "r"(parity), "r"(20000u)
            : "memory");
        if (done) return;
        if (spins > (1u << 22)) __trap();
    }
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    for (uint32_t spins = 0;; ++spins) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity), "r"(20000u)
            : "memory");
        if (done) return;
        if (spins > (1u << 22)) __trap();
    }
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            int w, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(bar))
        : "memory");
}

// The innermost box coordinate must be 16-byte aligned (measured: boxes
// starting at x0 - R fault with an illegal instruction unless 4R is a
// multiple of 16), so the a2 halo is widened to RA = R rounded up to 4.
template <int R, int NX>
struct TmaBox {
    static constexpr int RA = (R + 3) / 4 * 4;
    static constexpr int WB = 32 * NX + 2 * RA;  // 16-byte multiple rows
};

template <int R, int TY, int NX>
struct TmaLayout {
    static constexpr int RA = TmaBox<R, NX>::RA;
    static constexpr int WB = TmaBox<R, NX>::WB;
    static constexpr int H = TY + 2 * R;
    static constexpr int CUR_FLOATS = WB * H;
    static constexpr int CUR_BYTES = (CUR_FLOATS * 4 + 127) / 128 * 128;
    static constexpr int PME_FLOATS = 32 * NX * TY;
    static constexpr int PME_BYTES = (PME_FLOATS * 4 + 127) / 128 * 128;
    static constexpr int BAR_BYTES = 256;  // up to 31 stages + prologue barrier
    static constexpr size_t smem(int stages) {
        return BAR_BYTES + static_cast<size_t>(2 * R + stages) * CUR_BYTES +
               static_cast<size_t>(stages) * 3 * PME_BYTES;
    }
};

template <int R, bool FWD, int TY, int NX>
__global__ void __launch_bounds__(32 * TY) acoustic3d_tma_kernel(const __grid_constant__ TmaStencilArgs A) {
    using L = TmaLayout<R, TY, NX>;
    constexpr int WB = L::WB;
    constexpr int RA = L::RA;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    unsigned char* cur_base = smem + L::BAR_BYTES;
    const int S = A.stages;
    const int NR = 2 * R + S;
    unsigned char* pme_base = cur_base + static_cast<size_t>(NR) * L::CUR_BYTES;

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * 32 + tx;
    const int x0 = blockIdx.x * 32 * NX;
    const int y0 = blockIdx.y * TY;
    const int zb = A.z0 + blockIdx.z * A.zchunk;
    const int ze = min(zb + A.zchunk, A.z1);
    if (zb >= ze) return;  // uniform per CTA
    const int nit = ze - zb;

    auto cur_slot = [&](int p) {  // smem tile of cur plane p (zb-R <= p)
        return reinterpret_cast<float*>(cur_base + ((p - zb + R) % NR) * L::CUR_BYTES);
    };
    auto pme_slot = [&](int i, int f) {
        return reinterpret_cast<float*>(pme_base + ((i % S) * 3 + f) * L::PME_BYTES);
    };
    constexpr uint32_t group_bytes = L::CUR_FLOATS * 4 + 3 * L::PME_FLOATS * 4;
    auto issue_group = [&](int i) {
        uint64_t* b = &bar[i % S];
        const int z = zb + i;
        mbar_arrive_expect_tx(b, group_bytes);
        tma_load_4d(cur_slot(z + R), &A.cur, x0 - RA, y0 - R, z + R, A.lv_cur, b);
        tma_load_4d(pme_slot(i, 0), &A.prev, x0, y0, z, A.lv_prev, b);
        tma_load_4d(pme_slot(i, 1), &A.m, x0, y0, z, 0, b);
        tma_load_4d(pme_slot(i, 2), &A.eta, x0, y0, z, 0, b);
    };

    if (tid == 0) {
        for (int i = 0; i <= S; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        // prologue: planes zb-R .. zb+R-1 of cur on the extra barrier
        mbar_arrive_expect_tx(&bar[S], 2 * R * L::CUR_FLOATS * 4);
        for (int j = 0; j < 2 * R; ++j)
            tma_load_4d(cur_slot(zb - R + j), &A.cur, x0 - RA, y0 - R, zb - R + j, A.lv_cur, &bar[S]);
        for (int i = 0; i < S && i < nit; ++i) issue_group(i);
    }

    unsigned act = 0;
#pragma unroll
    for (int k = 0; k < NX; ++k) {
        const int a2 = x0 + tx + 32 * k;
        const int a1 = y0 + ty;
        if (a2 >= R && a2 < A.n2 - R && a1 >= R && a1 < A.n1 - R) act |= 1u << k;
    }
    const int cpos = (ty + R) * WB + tx + RA;  // centre of column k=0 in a cur tile
    const int ppos = ty * 32 * NX + tx;
    float* outp = A.out + static_cast<int64_t>(zb) * A.plane +
                  static_cast<int64_t>(y0 + ty) * A.pitch + x0 + tx;

    mbar_wait(&bar[S], 0);
    int ring0 = 0;              // ring slot of plane z-R  (= i mod NR)
    int stage = 0, phase = 0;   // i mod S, (i / S) & 1
    for (int i = 0; i < nit; ++i) {
        mbar_wait(&bar[stage], phase);
        const float* ring[2 * R + 1];  // tiles of planes z-R .. z+R
#pragma unroll
        for (int j = 0; j <= 2 * R; ++j) {
            int sl = ring0 + j;
            sl = sl >= NR ? sl - NR : sl;
            ring[j] = reinterpret_cast<const float*>(cur_base + sl * L::CUR_BYTES);
        }
        const float* pc = ring[R];
        const float* pp = reinterpret_cast<const float*>(pme_base + (stage * 3 + 0) * L::PME_BYTES);
        const float* pm = reinterpret_cast<const float*>(pme_base + (stage * 3 + 1) * L::PME_BYTES);
        const float* pe = reinterpret_cast<const float*>(pme_base + (stage * 3 + 2) * L::PME_BYTES);
#pragma unroll
        for (int k = 0; k < NX; ++k) {
            if (!(act & (1u << k))) continue;
            const int c = cpos + 32 * k;
            const float cv = pc[c];
            const float pv = pp[ppos + 32 * k];
            const float mv = pm[ppos + 32 * k];
            const float ev = pe[ppos + 32 * k];
            const float temp0 = __fmul_rn(A.ce, ev);
            const float temp1 = __fmul_rn(A.cm, mv);
            const float temp2 = __fadd_rn(temp0, temp1);
            const float temp3 = __fdiv_rn(1.0f, temp2);
            float acc;
            {
                acc = __fmul_rn(__fmul_rn(__fmul_rn(A.tc[0], temp3), ev), pv);
                if (FWD) {
                    acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(__fmul_rn(A.tc[1], temp3), mv), pv));
                    acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(__fmul_rn(A.tc[2], temp3), mv), cv));
                } else {
                    acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(__fmul_rn(A.tc[1], temp3), mv), cv));
                    acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(__fmul_rn(A.tc[2], temp3), mv), pv));
                }
            }
            acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(A.c0, temp3), cv));
            float kc[R];
#pragma unroll
            for (int j = 0; j < R; ++j) kc[j] = __fmul_rn(A.cj[j], temp3);
            // last axis (a2): offsets -R..-1, +1..+R
#pragma unroll
            for (int j = R; j >= 1; --j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], pc[c - j]));
#pragma unroll
            for (int j = 1; j <= R; ++j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], pc[c + j]));
            // axis 1
#pragma unroll
            for (int j = R; j >= 1; --j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], pc[c - j * WB]));
#pragma unroll
            for (int j = 1; j <= R; ++j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], pc[c + j * WB]));
            // axis 0: same position in the tiles of planes z-R..z+R
#pragma unroll
            for (int j = R; j >= 1; --j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], ring[R - j][c]));
#pragma unroll
            for (int j = 1; j <= R; ++j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], ring[R + j][c]));
            outp[32 * k] = acc;
        }
        outp += A.plane;
        __syncthreads();  // every thread is done with cur plane z-R and pme slot i
        if (tid == 0 && i + S < nit) issue_group(i + S);
        ring0 = ring0 + 1 == NR ? 0 : ring0 + 1;
        if (++stage == S) {
            stage = 0;
            phase ^= 1;
        }
    }
}

} // namespace sfb
