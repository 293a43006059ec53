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
// 2.5D scheme: a CTA owns a 32 x TY tile of (a2, a1) columns and streams
// along a0 (the slowest axis, depth) over zchunk planes. Each thread keeps
// the 2R+1 values of its own column along a0 in a register queue, so the a0
// neighbours cost one coalesced load per plane; the current plane plus
// R-wide a2/a1 halos are staged in shared memory for the in-plane
// neighbours. Per point the compulsory DRAM traffic is cur + prev + m + eta
// reads and one write (20 B); halo re-reads are served by L2.
// GRAD (FWI adjoint): before overwriting the output slot (which holds
// v(t+2)) accumulate grad += u(t+1) * ((v(t+2) - 2 v(t+1)) + v(t)) * cm.
template <int R, bool FWD, int TY, bool GRAD>
__global__ void __launch_bounds__(32 * TY)
acoustic3d_kernel(const StencilArgs A) {
    __shared__ float s[TY + 2 * R][32 + 2 * R];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int a2 = blockIdx.x * 32 + tx;
    const int a1 = blockIdx.y * TY + ty;
    const int zb = R + blockIdx.z * A.zchunk;
    const int ze = min(zb + A.zchunk, A.n0 - R);
    if (zb >= ze) return;  // uniform per CTA
    const bool in_arr = a2 < A.n2 && a1 < A.n1;
    const bool active = in_arr && a2 >= R && a2 < A.n2 - R && a1 >= R && a1 < A.n1 - R;
    const int64_t col = static_cast<int64_t>(a1) * A.pitch + a2;

    float q[2 * R + 1];
#pragma unroll
    for (int k = 0; k < 2 * R; ++k)
        q[k + 1] = in_arr ? __ldg(A.cur + static_cast<int64_t>(zb - R + k) * A.plane + col) : 0.0f;

    // halo sources for this thread (fixed across planes)
    const int hl = blockIdx.x * 32 - R + tx;     // a2 of left halo (tx < R)
    const int hr = blockIdx.x * 32 + 32 + tx;    // a2 of right halo (tx < R)
    const int vl = blockIdx.y * TY - R + ty;     // a1 of lower halo (ty < R)
    const int vr = blockIdx.y * TY + TY + ty;    // a1 of upper halo (ty < R)
    const bool do_hl = tx < R && a1 < A.n1 && hl >= 0;
    const bool do_hr = tx < R && a1 < A.n1 && hr < A.n2;
    const bool do_vl = ty < R && a2 < A.n2 && vl >= 0;
    const bool do_vr = ty < R && a2 < A.n2 && vr < A.n1;
    const int64_t off_hl = static_cast<int64_t>(a1) * A.pitch + hl;
    const int64_t off_hr = static_cast<int64_t>(a1) * A.pitch + hr;
    const int64_t off_vl = static_cast<int64_t>(vl) * A.pitch + a2;
    const int64_t off_vr = static_cast<int64_t>(vr) * A.pitch + a2;

    for (int z = zb; z < ze; ++z) {
#pragma unroll
        for (int k = 0; k < 2 * R; ++k) q[k] = q[k + 1];
        const int64_t pz = static_cast<int64_t>(z) * A.plane;
        q[2 * R] = in_arr ? __ldg(A.cur + pz + static_cast<int64_t>(R) * A.plane + col) : 0.0f;
        float pv = 0.0f, mv = 0.0f, ev = 0.0f, old = 0.0f, uh = 0.0f, gv = 0.0f;
        if (active) {
            pv = __ldg(A.prev + pz + col);
            mv = __ldg(A.m + pz + col);
            ev = __ldg(A.eta + pz + col);
            if (GRAD) {
                old = A.out[pz + col];
                uh = __ldg(A.uhist + pz + col);
                gv = A.grad[pz + col];
            }
        }
        const float hlv = do_hl ? __ldg(A.cur + pz + off_hl) : 0.0f;
        const float hrv = do_hr ? __ldg(A.cur + pz + off_hr) : 0.0f;
        const float vlv = do_vl ? __ldg(A.cur + pz + off_vl) : 0.0f;
        const float vrv = do_vr ? __ldg(A.cur + pz + off_vr) : 0.0f;
        __syncthreads();  // previous plane fully consumed
        s[ty + R][tx + R] = q[R];
        if (tx < R) {
            s[ty + R][tx] = hlv;
            s[ty + R][tx + 32 + R] = hrv;
        }
        if (ty < R) {
            s[ty][tx + R] = vlv;
            s[ty + TY + R][tx + R] = vrv;
        }
        __syncthreads();
        if (active) {
            const float cv = q[R];
            const float temp0 = __fmul_rn(A.ce, ev);
            const float temp1 = __fmul_rn(A.cm, mv);
            const float temp2 = __fadd_rn(temp0, temp1);
            const float temp3 = __fdiv_rn(1.0f, temp2);
            float acc = time_terms<FWD>(A, temp3, ev, mv, pv, cv);
            acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(A.c0, temp3), cv));
            float kc[R];
#pragma unroll
            for (int j = 0; j < R; ++j) kc[j] = __fmul_rn(A.cj[j], temp3);
            // last axis (a2): offsets -R..-1, +1..+R
#pragma unroll
            for (int j = R; j >= 1; --j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], s[ty + R][tx + R - j]));
#pragma unroll
            for (int j = 1; j <= R; ++j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], s[ty + R][tx + R + j]));
            // axis 1
#pragma unroll
            for (int j = R; j >= 1; --j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], s[ty + R - j][tx + R]));
#pragma unroll
            for (int j = 1; j <= R; ++j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], s[ty + R + j][tx + R]));
            // axis 0 (register queue)
#pragma unroll
            for (int j = R; j >= 1; --j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], q[R - j]));
#pragma unroll
            for (int j = 1; j <= R; ++j) acc = __fadd_rn(acc, __fmul_rn(kc[j - 1], q[R + j]));
            if (GRAD) {
                const float vtt = __fmul_rn(__fadd_rn(__fsub_rn(old, __fmul_rn(2.0f, pv)), cv), A.cm);
                A.grad[pz + col] = __fadd_rn(gv, __fmul_rn(uh, vtt));
            }
            A.out[pz + col] = acc;
        }
    }
}

// ---------------------------------------------------------------------------
// 2D acoustic update (parity/adjoint-test sizes): one thread per point,
// neighbours through the read-only cache. Axes: a0 (slow), a1 (contiguous).
template <int R, bool FWD>
__global__ void __launch_bounds__(256) acoustic2d_kernel(const StencilArgs A) {
    const int a1 = blockIdx.x * blockDim.x + threadIdx.x;
    const int a0 = blockIdx.y * blockDim.y + threadIdx.y;
    if (a1 < R || a1 >= A.n1 - R || a0 < R || a0 >= A.n0 - R) return;
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
};

__global__ void __launch_bounds__(256) inject_kernel(const InjectArgs A) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.ncells) return;
    const int64_t off = A.cell_off[i];
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
};

template <int NDIM>
__global__ void __launch_bounds__(256) sample_kernel(const SampleArgs A) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= A.np) return;
    constexpr int C = 1 << NDIM;
    const int c0 = A.ci[p * NDIM + 0];
    const int c1 = A.ci[p * NDIM + 1];
    const int c2 = NDIM == 3 ? A.ci[p * NDIM + 2] : 0;
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
