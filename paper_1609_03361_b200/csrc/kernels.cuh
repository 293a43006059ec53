// kernels.cuh — sm_100a kernels of the stencil hot path.
//
// Arithmetic contract: every kernel reproduces, operation for operation, the
// fp32 expression the reference emits for the same update (golden
// tests/golden/acoustic_3d.c:35-39, diffusion_1000.c:23, injection
// acoustic_3d.c:43-54, sampling acoustic_3d.c:55-59): products evaluated left
// to right, sums left to right, no FMA contraction (the reference compiles
// with -ffp-contract=off, jit.cpp:70), IEEE division, denormals preserved.
// The explicit __fmul_rn/__fadd_rn/__fdiv_rn intrinsics pin that order no
// matter what nvcc's contraction flags are; the library is also built with
// --fmad=false and without fast-math.
//
// Layout in HBM: each field is stored with its contiguous axis padded to a
// multiple of 32 floats (128-byte rows): off(a0,a1,a2) = a0*plane + a1*pitch
// + a2, plane = n1*pitch (3D); off(a0,a1) = a0*pitch + a1 (2D). Interior
// points are [r, n-r) on every axis (ir.cpp:198-199); the boundary strip is
// never written by the stencil.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sfb {

struct StencilArgs {
    float* out;
    const float* cur;
    const float* prev;
    const float* m;
    const float* eta;
    float* grad;         // FWI: gradient accumulator (GRAD kernels only)
    const float* uhist;  // FWI: forward level u(t+1) for the delayed gradient term
    int64_t pitch;       // row pitch (elements)
    int64_t plane;       // plane stride (elements, 3D)
    int n0, n1, n2;
    int zchunk;          // planes of axis 0 per block (3D)
    int z0, z1;          // planes of axis 0 this launch updates (interior, or a slab's)
    float ce, cm;
    float tc[3];
    float c0;
    float cj[8];
};

// The three time terms in emitted order (see acoustic_constants()):
//   forward: tc0*t3*eta*prev + tc1*t3*m*prev + tc2*t3*m*cur
//   adjoint: tc0*t3*eta*prev + tc1*t3*m*cur  + tc2*t3*m*prev
template <bool FWD>
__device__ __forceinline__ float time_terms(const StencilArgs& A, float temp3, float ev, float mv,
                                            float pv, float cv) {
    float acc = __fmul_rn(__fmul_rn(__fmul_rn(A.tc[0], temp3), ev), pv);
    if (FWD) {
        acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(__fmul_rn(A.tc[1], temp3), mv), pv));
        acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(__fmul_rn(A.tc[2], temp3), mv), cv));
    } else {
        acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(__fmul_rn(A.tc[1], temp3), mv), cv));
        acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(__fmul_rn(A.tc[2], temp3), mv), pv));
    }
    return acc;
}

// ---------------------------------------------------------------------------
// K2/K3: 3D acoustic forward/adjoint update, space order 2R.
//
// 2.5D scheme. A CTA of 32 x TY threads owns a (32*NX) x TY tile of
// (a2, a1) columns and streams along a0 (the slowest axis, depth) over
// zchunk planes. Thread (tx, ty) owns the NX columns a2 = x0 + tx + 32k,
// k < NX: every global access of a warp is one fully coalesced 128-byte
// line and the NX accesses of a thread share one address (immediate
// offsets), which amortises address arithmetic over NX points.
//  * a0 neighbours: each thread keeps the 2R+1 values of its columns along
//    a0 in a register queue (one new load per plane);
//  * a2/a1 neighbours: the current plane plus R-wide halos is staged in a
//    double-buffered shared-memory tile (one __syncthreads per plane);
//  * the loads for plane z+1 (queue head, u(t-1), m, eta, halos) are issued
//    before plane z is computed (two register sets, loop unrolled by two),
//    so a whole plane of math hides their latency.
// Addressing is 32-bit element offsets from the field bases (fields are
// < 2^31 elements), advanced by one plane per step. Fields are allocated
// with guard slack after the last plane (alloc_field), so every tile load
// is in bounds and unpredicated; only the stores are masked to the
// interior. Compulsory DRAM traffic per point: u(t), u(t-1), m, eta reads
// and the u(t+1) write = 20 B; halo re-reads hit L2.
// GRAD (FWI adjoint): before overwriting the output slot (which holds
// v(t+2)) accumulate grad += u(t+1) * ((v(t+2) - 2 v(t+1)) + v(t)) * cm.
template <int NX, bool GRAD>
struct PlaneRegs {
    float q[NX], pv[NX], mv[NX], ev[NX], vl[NX], vr[NX], h;
    float old[NX], uh[NX], gv[NX];
};

template <int R, bool FWD, int TY, int NX, bool GRAD>
__global__ void __launch_bounds__(32 * TY)
acoustic3d_kernel(const StencilArgs A) {
    constexpr int W = 32 * NX + 2 * R;  // smem row length
    constexpr int H = TY + 2 * R;
    __shared__ float s[2][H][W];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int x0 = blockIdx.x * 32 * NX;
    const int a1 = blockIdx.y * TY + ty;
    const int zb = A.z0 + blockIdx.z * A.zchunk;
    const int ze = min(zb + A.zchunk, A.z1);
    if (zb >= ze) return;  // uniform per CTA

    const int pitch = static_cast<int>(A.pitch);
    const int plane = static_cast<int>(A.plane);
    unsigned act = 0;  // bit k: column k is an interior point
#pragma unroll
    for (int k = 0; k < NX; ++k) {
        const int a2 = x0 + tx + 32 * k;
        if (a2 >= R && a2 < A.n2 - R && a1 >= R && a1 < A.n1 - R) act |= 1u << k;
    }
    // halo roles: lanes tx < R load the left a2 halo, lanes tx >= 32-R the
    // right one (row a1); warps ty < R load the a1 halo rows of the tile
    const bool hl = tx < R, hr = tx >= 32 - R, vh = ty < R;
    const int hxo = hl ? (-R) : (32 * NX - (32 - R));  // a2 offset of this lane's halo
    const int col = a1 * pitch + x0 + tx;
    // element offsets relative to `col` of the halo loads of this thread
    const int o_vl = (blockIdx.y * TY - R + ty - a1) * pitch;   // row a1-halo below
    const int o_vr = (blockIdx.y * TY + TY + ty - a1) * pitch;  // row a1-halo above
    const int o_h = hxo;                                         // same row, a2 halo

    float q[NX][2 * R + 1];
    int off = (zb - R) * plane + col;  // offset of plane (zb - R) at this column
#pragma unroll
    for (int j = 0; j < 2 * R; ++j) {
#pragma unroll
        for (int k = 0; k < NX; ++k) q[k][j + 1] = __ldg(A.cur + off + 32 * k);
        off += plane;
    }
    // now off = offset of plane zb + R (the next queue head)

    auto prefetch = [&](PlaneRegs<NX, GRAD>& P, int o /* plane z at col */) {
        const float* c = A.cur + o;
        const float* qh = A.cur + (o + R * plane);
        const float* pp = A.prev + o;
        const float* mp = A.m + o;
        const float* ep = A.eta + o;
#pragma unroll
        for (int k = 0; k < NX; ++k) {
            P.q[k] = __ldg(qh + 32 * k);
            P.pv[k] = __ldg(pp + 32 * k);
            P.mv[k] = __ldg(mp + 32 * k);
            P.ev[k] = __ldg(ep + 32 * k);
        }
        if (GRAD) {
            const float* op = A.out + o;
            const float* up = A.uhist + o;
            const float* gp = A.grad + o;
#pragma unroll
            for (int k = 0; k < NX; ++k) {
                P.old[k] = op[32 * k];
                P.uh[k] = __ldg(up + 32 * k);
                P.gv[k] = gp[32 * k];
            }
        }
        if (vh) {
#pragma unroll
            for (int k = 0; k < NX; ++k) {
                P.vl[k] = __ldg(c + o_vl + 32 * k);
                P.vr[k] = __ldg(c + o_vr + 32 * k);
            }
        }
        if (hl || hr) P.h = __ldg(c + o_h);
    };

    auto step = [&](PlaneRegs<NX, GRAD>& P, PlaneRegs<NX, GRAD>& Nx, int z, int o,
                    float (*sb)[W]) {
#pragma unroll
        for (int k = 0; k < NX; ++k) {
#pragma unroll
            for (int j = 0; j < 2 * R; ++j) q[k][j] = q[k][j + 1];
            q[k][2 * R] = P.q[k];
            sb[ty + R][tx + R + 32 * k] = q[k][R];
        }
        if (vh) {
#pragma unroll
            for (int k = 0; k < NX; ++k) {
                sb[ty][tx + R + 32 * k] = P.vl[k];
                sb[ty + TY + R][tx + R + 32 * k] = P.vr[k];
            }
        }
        if (hl || hr) sb[ty + R][tx + R + hxo] = P.h;
        __syncthreads();
        if (z + 1 < ze) prefetch(Nx, o + plane);
#pragma unroll
        for (int k = 0; k < NX; ++k) {
            if (!(act & (1u << k))) continue;
            const float cv = q[k][R];
            const float temp0 = __fmul_rn(A.ce, P.ev[k]);
            const float temp1 = __fmul_rn(A.cm, P.mv[k]);
            const float temp2 = __fadd_rn(temp0, temp1);
            const float temp3 = __fdiv_rn(1.0f, temp2);
            float acc = time_terms<FWD>(A, temp3, P.ev[k], P.mv[k], P.pv[k], cv);
            acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(A.c0, temp3), cv));
            float kc[R];
#pragma unroll
            for (int j = 0; j < R; ++j) kc[j] = __fmul_rn(A.cj[j], temp3);
            const float* row = &sb[ty + R][tx + R + 32 * k];
            // last axis (a2): offsets -R..-1, +1..+R
#pragma unroll
            for (int j = R; j >= 1; --j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], row[-j]));
#pragma unroll
            for (int j = 1; j <= R; ++j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], row[j]));
            // axis 1
#pragma unroll
            for (int j = R; j >= 1; --j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], row[-j * W]));
#pragma unroll
            for (int j = 1; j <= R; ++j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], row[j * W]));
            // axis 0 (register queue)
#pragma unroll
            for (int j = R; j >= 1; --j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], q[k][R - j]));
#pragma unroll
            for (int j = 1; j <= R; ++j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], q[k][R + j]));
            if (GRAD) {
                const float vtt = __fmul_rn(
                    __fadd_rn(__fsub_rn(P.old[k], __fmul_rn(2.0f, P.pv[k])), cv), A.cm);
                A.grad[o + 32 * k] = __fadd_rn(P.gv[k], __fmul_rn(P.uh[k], vtt));
            }
            A.out[o + 32 * k] = acc;
        }
    };

    PlaneRegs<NX, GRAD> P0, P1;
    int o = zb * plane + col;
    prefetch(P0, o);
    for (int z = zb; z < ze; z += 2) {
        step(P0, P1, z, o, s[0]);
        o += plane;
        if (z + 1 < ze) step(P1, P0, z + 1, o, s[1]);
        o += plane;
    }
}

// ---------------------------------------------------------------------------
// 2D acoustic update (parity/adjoint-test sizes): one thread per point,
// neighbours through the read-only cache. Axes: a0 (slow), a1 (contiguous).
template <int R, bool FWD>
__global__ void __launch_bounds__(256) acoustic2d_kernel(const StencilArgs A) {
    const int a1 = blockIdx.x * blockDim.x + threadIdx.x;
    const int a0 = blockIdx.y * blockDim.y + threadIdx.y;
    if (a1 < R || a1 >= A.n1 - R || a0 < A.z0 || a0 >= A.z1) return;
    const int64_t o = static_cast<int64_t>(a0) * A.pitch + a1;
    const float* c = A.cur + o;
    const float ev = __ldg(A.eta + o), mv = __ldg(A.m + o), pv = __ldg(A.prev + o), cv = __ldg(c);
    const float temp0 = __fmul_rn(A.ce, ev);
    const float temp1 = __fmul_rn(A.cm, mv);
    const float temp2 = __fadd_rn(temp0, temp1);
    const float temp3 = __fdiv_rn(1.0f, temp2);
    float acc = time_terms<FWD>(A, temp3, ev, mv, pv, cv);
    acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(A.c0, temp3), cv));
    float kc[R];
#pragma unroll
    for (int j = 0; j < R; ++j) kc[j] = __fmul_rn(A.cj[j], temp3);
#pragma unroll
    for (int j = R; j >= 1; --j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], __ldg(c - j)));
#pragma unroll
    for (int j = 1; j <= R; ++j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], __ldg(c + j)));
#pragma unroll
    for (int j = R; j >= 1; --j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], __ldg(c - j * A.pitch)));
#pragma unroll
    for (int j = 1; j <= R; ++j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], __ldg(c + j * A.pitch)));
    A.out[o] = acc;
}

// ---------------------------------------------------------------------------
// K4: deterministic source injection. The reference runs the 2^d corner
// updates of every point sequentially in p order (omp single, ir.cpp:359):
//   f[c] = ((scale*series[p])*w[p][k])/m[c] + f[c]
// Collisions are resolved exactly by a host-built CSR over the distinct
// target cells: one thread per cell applies that cell's contributions in
// ascending p, which is the reference's sequence restricted to that cell.
struct InjectArgs {
    float* field;
    const float* m;
    const float* row;         // series row of this step: series + row_index*np
    const int64_t* cell_off;  // distinct target cells (device offsets)
    const int* start;         // [ncells+1] contribution ranges
    const int* cp;            // contribution point index p
    const float* cw;          // contribution weight w[p][k]
    float scale;
    int ncells;
    // plane filter (time-skewed steps, plan.cu invoke_overlapped): when
    // zf1 > 0 only cells whose a0 plane lies in [zf0, zf1) are injected
    int64_t plane;
    int zf0, zf1;
};

__global__ void __launch_bounds__(256) inject_kernel(const InjectArgs A) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.ncells) return;
    const int64_t off = A.cell_off[i];
    if (A.zf1 > 0) {
        const int z = static_cast<int>(off / A.plane);
        if (z < A.zf0 || z >= A.zf1) return;
    }
    float v = A.field[off];
    const float mv = __ldg(A.m + off);
    for (int j = A.start[i]; j < A.start[i + 1]; ++j) {
        const float d = __fdiv_rn(__fmul_rn(__fmul_rn(A.scale, __ldg(A.row + A.cp[j])), A.cw[j]), mv);
        v = __fadd_rn(d, v);
    }
    A.field[off] = v;
}

// ---------------------------------------------------------------------------
// K5: receiver interpolation, one thread per point:
//   out[p] = w0*f[c0] + w1*f[c1] + ... (corner k: bit i adds +1 on axis i).
struct SampleArgs {
    const float* field;
    const int* ci;     // [np][ndim]
    const float* w;    // [np][2^ndim]
    float* out;        // series row of this step
    int64_t pitch, plane;
    int np;
    // plane filter (time-skewed steps): when zf1 > 0 only points whose upper
    // corner plane c0 + 1 lies in [zf0, zf1) are sampled
    int zf0, zf1;
};

template <int NDIM>
__global__ void __launch_bounds__(256) sample_kernel(const SampleArgs A) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= A.np) return;
    constexpr int C = 1 << NDIM;
    const int c0 = A.ci[p * NDIM + 0];
    const int c1 = A.ci[p * NDIM + 1];
    const int c2 = NDIM == 3 ? A.ci[p * NDIM + 2] : 0;
    if (A.zf1 > 0 && (c0 + 1 < A.zf0 || c0 + 1 >= A.zf1)) return;
    float acc = 0.0f;
#pragma unroll
    for (int k = 0; k < C; ++k) {
        int64_t off;
        if (NDIM == 3)
            off = static_cast<int64_t>(c0 + (k & 1)) * A.plane +
                  static_cast<int64_t>(c1 + ((k >> 1) & 1)) * A.pitch + (c2 + ((k >> 2) & 1));
        else
            off = static_cast<int64_t>(c0 + (k & 1)) * A.pitch + (c1 + ((k >> 1) & 1));
        const float term = __fmul_rn(A.w[p * C + k], A.field[off]);
        acc = k == 0 ? term : __fadd_rn(acc, term);
    }
    A.out[p] = acc;
}

// ---------------------------------------------------------------------------
// K4+K5 fused for small point sets (one CTA): injection into the distinct
// target cells, a CTA barrier, then sampling — the reference's two
// sequential `omp single` loops (golden acoustic_3d.c:43-59) in one launch.
template <int NDIM>
__global__ void __launch_bounds__(1024) inject_sample_kernel(const InjectArgs I, const SampleArgs S) {
    for (int i = threadIdx.x; i < I.ncells; i += blockDim.x) {
        const int64_t off = I.cell_off[i];
        float v = I.field[off];
        const float mv = __ldg(I.m + off);
        for (int j = I.start[i]; j < I.start[i + 1]; ++j) {
            const float d =
                __fdiv_rn(__fmul_rn(__fmul_rn(I.scale, __ldg(I.row + I.cp[j])), I.cw[j]), mv);
            v = __fadd_rn(d, v);
        }
        I.field[off] = v;
    }
    __syncthreads();  // orders the injected stores before the samples' loads (CTA scope)
    constexpr int C = 1 << NDIM;
    for (int p = threadIdx.x; p < S.np; p += blockDim.x) {
        const int c0 = S.ci[p * NDIM + 0];
        const int c1 = S.ci[p * NDIM + 1];
        const int c2 = NDIM == 3 ? S.ci[p * NDIM + 2] : 0;
        float acc = 0.0f;
#pragma unroll
        for (int k = 0; k < C; ++k) {
            int64_t off;
            if (NDIM == 3)
                off = static_cast<int64_t>(c0 + (k & 1)) * S.plane +
                      static_cast<int64_t>(c1 + ((k >> 1) & 1)) * S.pitch + (c2 + ((k >> 2) & 1));
            else
                off = static_cast<int64_t>(c0 + (k & 1)) * S.pitch + (c1 + ((k >> 1) & 1));
            const float term = __fmul_rn(S.w[p * C + k], S.field[off]);
            acc = k == 0 ? term : __fadd_rn(acc, term);
        }
        S.out[p] = acc;
    }
}

// ---------------------------------------------------------------------------
// Host-boundary repack between the reference's dense rows (width floats) and
// the padded HBM rows (pitch floats): the H2D/D2H copies themselves are then
// single contiguous transfers at full PCIe speed.
__global__ void __launch_bounds__(256)
repack_rows_kernel(float* __restrict__ dst, int64_t dst_pitch, const float* __restrict__ src,
                   int64_t src_pitch, int64_t rows, int width) {
    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        const float* s = src + row * src_pitch;
        float* d = dst + row * dst_pitch;
        for (int c = threadIdx.x; c < width; c += blockDim.x) d[c] = s[c];
    }
}

// ---------------------------------------------------------------------------
// FWI: the gradient term for time t = 1 after the adjoint sweep
// (grad += u(1) * ((v(2) - 2 v(1)) + v(0)) * cm on the interior).
__global__ void __launch_bounds__(256)
grad_final_kernel(float* grad, const float* u1, const float* v2, const float* v1, const float* v0,
                  float cm, int64_t pitch, int64_t plane, int n0, int n1, int n2, int r) {
    const int a2 = blockIdx.x * blockDim.x + threadIdx.x;
    const int a1 = blockIdx.y;
    const int a0 = blockIdx.z;
    if (a2 < r || a2 >= n2 - r || a1 < r || a1 >= n1 - r || a0 < r || a0 >= n0 - r) return;
    const int64_t o = static_cast<int64_t>(a0) * plane + static_cast<int64_t>(a1) * pitch + a2;
    const float vtt = __fmul_rn(__fadd_rn(__fsub_rn(v2[o], __fmul_rn(2.0f, v1[o])), v0[o]), cm);
    grad[o] = __fadd_rn(grad[o], __fmul_rn(u1[o], vtt));
}

// ---------------------------------------------------------------------------
// K1: diffusion update, any order: out = c0*u + sum (last axis first,
// offsets -R..-1, +1..+R) cj*u[nbr], left to right; the centre term is
// absent when its folded coefficient is exactly zero (order 2 at the
// stability limit, golden diffusion_1000.c:23).
struct DiffusionArgs {
    float* out;
    const float* cur;
    int64_t pitch;
    int n0, n1;
    float c0;
    int has_c0;
    float cj[8];
};

template <int R>
__global__ void __launch_bounds__(256) diffusion_kernel(const DiffusionArgs A) {
    const int a1 = blockIdx.x * blockDim.x + threadIdx.x;
    const int a0 = blockIdx.y * blockDim.y + threadIdx.y;
    if (a1 < R || a1 >= A.n1 - R || a0 < R || a0 >= A.n0 - R) return;
    const int64_t o = static_cast<int64_t>(a0) * A.pitch + a1;
    const float* c = A.cur + o;
    float acc;
    bool first = true;
    if (A.has_c0) {
        acc = __fmul_rn(A.c0, __ldg(c));
        first = false;
    }
#pragma unroll
    for (int j = R; j >= 1; --j) {
        const float t = __fmul_rn(A.cj[j - 1], __ldg(c - j));
        acc = first ? t : __fadd_rn(acc, t);
        first = false;
    }
#pragma unroll
    for (int j = 1; j <= R; ++j) acc = __fadd_rn(acc, __fmul_rn(A.cj[j - 1], __ldg(c + j)));
#pragma unroll
    for (int j = R; j >= 1; --j) acc = __fadd_rn(acc, __fmul_rn(A.cj[j - 1], __ldg(c - j * A.pitch)));
#pragma unroll
    for (int j = 1; j <= R; ++j) acc = __fadd_rn(acc, __fmul_rn(A.cj[j - 1], __ldg(c + j * A.pitch)));
    A.out[o] = acc;
}

} // namespace sfb
