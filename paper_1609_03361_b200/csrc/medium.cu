// medium.cu — seeded smooth random velocity media on the device (SURVEY
// 8(d): configs C3, C4, C5 use "smooth random v in [1.5, 4.5] km/s from
// seeded Gaussian-filtered noise (sigma = 8 cells)").
//
// Definition (restated in C by oracle/sf_port.c sfp_smooth_* for the tests):
//   noise(i)  = uniform in [-1, 1) on a 2^-23 lattice from a splitmix64 hash
//               of the GLOBAL linear cell index i and the seed, so any slab
//               of a decomposed grid generates its planes without the rest;
//   g[k]      = exp(-x^2 / (2 sigma^2)), x = k - rad, rad = int(4 sigma + 0.5),
//               normalised to unit sum (host, double);
//   t1        = float(sum_k g[k] * noise(i0, i1, refl(i2 + x)))     (axis 2)
//   t2        = float(sum_k g[k] * t1(i0, refl(i1 + x), i2))        (axis 1)
//   f         = sum_k g[k] * t2(refl(i0 + x), i1, i2)   (double, axis 0)
//               every sum in double, ascending k, no contraction;
//               refl = mirror about the faces (scipy.ndimage mode "reflect");
//   v         = v_lo + ((v_hi - v_lo) * (f - lo)) / (hi - lo), with lo/hi the
//               extrema of f over the whole GLOBAL grid (slabs combine their
//               own extrema with a min/max reduction);
//   m, eta    = build_medium's per-cell expressions (acoustic.cpp:67-105,
//               sfb::build_medium): m = float(1/(v*v)), eta = float(mv*sigma)
//               with sigma from the global distance to the nearest face.
// Pass 1 (mode EXTREMA) returns lo/hi of the requested planes; pass 2 (mode
// WRITE) recomputes f and writes m/eta with the caller's row/plane strides
// (dense host staging or a plan's padded HBM fields).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "medium.h"

namespace sfb {
namespace {

#define MED_CUDA(expr)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            throw MediumError(e_ == cudaErrorMemoryAllocation ? 1 : 2,                  \
                              std::string(#expr) + ": " + cudaGetErrorString(e_));      \
    } while (0)

struct Taps {
    double g[2 * kMediumMaxRad + 1];
    int rad;
};

__host__ __device__ __forceinline__ int64_t reflect_index(int64_t i, int64_t n) {
    const int64_t p = 2 * n;
    i %= p;
    if (i < 0) i += p;
    return i < n ? i : p - 1 - i;
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double noise_at(uint64_t salt, int64_t lin) {
    const uint64_t z = mix64(static_cast<uint64_t>(lin) * 0x9E3779B97F4A7C15ull + salt);
    return static_cast<double>(static_cast<int64_t>(z >> 40) - 8388608) * (1.0 / 8388608.0);
}

unsigned grid_for(int64_t n) {
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)));
}

// t1 over planes [L, L + nz) (axis-2 filter of the hashed noise)
__global__ void smooth_rows_kernel(float* __restrict__ t1, int64_t L, int64_t nz, int64_t n1,
                                   int64_t n2, uint64_t salt, const Taps T) {
    const int64_t total = nz * n1 * n2;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i2 = i % n2;
        const int64_t r = i / n2;  // (i0 - L) * n1 + i1
        const int64_t rowlin = (r + L * n1) * n2;  // global linear index of (i0, i1, 0)
        double s = 0.0;
        for (int k = 0; k <= 2 * T.rad; ++k)
            s = __dadd_rn(s, __dmul_rn(T.g[k], noise_at(salt, rowlin + reflect_index(i2 + k - T.rad, n2))));
        t1[i] = __double2float_rn(s);
    }
}

// t2 = axis-1 filter of t1 (same plane range)
__global__ void smooth_cols_kernel(float* __restrict__ t2, const float* __restrict__ t1, int64_t nz,
                                   int64_t n1, int64_t n2, const Taps T) {
    const int64_t total = nz * n1 * n2;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i2 = i % n2;
        const int64_t i1 = (i / n2) % n1;
        const int64_t base = i - i1 * n2;
        double s = 0.0;
        for (int k = 0; k <= 2 * T.rad; ++k)
            s = __dadd_rn(s, __dmul_rn(T.g[k], static_cast<double>(
                                                   __ldg(t1 + base + reflect_index(i1 + k - T.rad, n1) * n2))));
        t2[i] = __double2float_rn(s);
    }
}

// order-preserving key of a double (for atomicMin / atomicMax)
__device__ __forceinline__ unsigned long long dkey(double v) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

struct DepthArgs {
    const float* t2;
    int64_t L, n0, n1, n2;   // t2 holds global planes [L, ...); n0 global
    int64_t b, e;            // global planes to produce
    int64_t gn1, gn2;        // == n1, n2
    unsigned long long* ext; // [2] keys: min, max   (mode 0)
    float* m;                // mode 1 outputs, plane b at offset 0
    float* eta;
    int64_t pitch, plane;
    double lo, hi, v_lo, v_hi;
    int bw;
    int mode;
};

__global__ void smooth_depth_kernel(const DepthArgs A, const Taps T, const double* __restrict__ sig) {
    const int64_t n12 = A.n1 * A.n2;
    const int64_t total = (A.e - A.b) * n12;
    double mn = INFINITY, mx = -INFINITY;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t rest = i % n12;
        const int64_t i0 = A.b + i / n12;
        double f = 0.0;
        for (int k = 0; k <= 2 * T.rad; ++k)
            f = __dadd_rn(f, __dmul_rn(T.g[k], static_cast<double>(__ldg(
                                                   A.t2 + (reflect_index(i0 + k - T.rad, A.n0) - A.L) * n12 + rest))));
        if (A.mode == 0) {
            mn = fmin(mn, f);
            mx = fmax(mx, f);
            continue;
        }
        const int64_t i1 = rest / A.n2, i2 = rest % A.n2;
        const double v = __dadd_rn(A.v_lo, __ddiv_rn(__dmul_rn(__dsub_rn(A.v_hi, A.v_lo), __dsub_rn(f, A.lo)),
                                                     __dsub_rn(A.hi, A.lo)));
        const double mv = __ddiv_rn(1.0, __dmul_rn(v, v));
        int64_t dist = A.n0;
        dist = min(dist, i0);
        dist = min(dist, A.n0 - 1 - i0);
        dist = min(dist, i1);
        dist = min(dist, A.n1 - 1 - i1);
        dist = min(dist, i2);
        dist = min(dist, A.n2 - 1 - i2);
        const double sigma = (A.bw > 0 && dist < A.bw) ? sig[dist] : 0.0;
        const int64_t off = (i0 - A.b) * A.plane + i1 * A.pitch + i2;
        A.m[off] = __double2float_rn(mv);
        A.eta[off] = __double2float_rn(__dmul_rn(mv, sigma));
    }
    if (A.mode == 0) {
        for (int o = 16; o > 0; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(A.ext + 0, dkey(mn));
            atomicMax(A.ext + 1, dkey(mx));
        }
    }
}

double key_to_double(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double v;
    std::memcpy(&v, &b, sizeof v);
    return v;
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    explicit DevBuf(size_t n) { MED_CUDA(cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1))); }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

} // namespace

int smooth_radius(double sigma) { return static_cast<int>(4.0 * sigma + 0.5); }

std::vector<double> smooth_taps(double sigma) {
    const int rad = smooth_radius(sigma);
    std::vector<double> g(2 * rad + 1);
    double sum = 0.0;
    for (int k = 0; k <= 2 * rad; ++k) {
        const double x = static_cast<double>(k - rad);
        g[k] = std::exp(-0.5 * x * x / (sigma * sigma));
        sum += g[k];
    }
    for (double& v : g) v /= sum;
    return g;
}

uint64_t smooth_salt(uint64_t seed) { return mix64(seed + 0x9E3779B97F4A7C15ull); }

std::vector<double> sponge_sigma(int boundary_width, double spacing, double v_min) {
    // build_medium (acoustic.cpp:67-105): sigma(dist) for dist < w
    const long w = boundary_width;
    const double sigma_max =
        1.5 * std::log(1000.0) * v_min / (static_cast<double>(std::max<long>(w, 1)) * spacing);
    std::vector<double> s(std::max<long>(w, 1), 0.0);
    for (long d = 0; d < w; ++d) {
        const double rr = 1.0 - static_cast<double>(d) / static_cast<double>(w);
        s[d] = sigma_max * rr * rr;
    }
    return s;
}

void smooth_medium_run(const sf_smooth_medium_desc& d, int mode, double* lo, double* hi,
                       float* m, float* eta, int64_t pitch, int64_t plane, cudaStream_t st) {
    const int64_t n0 = d.shape[0], n1 = d.shape[1], n2 = d.shape[2];
    if (n0 < 1 || n1 < 1 || n2 < 1) throw MediumError(0, "smooth medium: empty grid");
    if (d.a0_begin < 0 || d.a0_end > n0 || d.a0_begin >= d.a0_end)
        throw MediumError(0, "smooth medium: plane range outside the grid");
    if (!(d.sigma > 0) || smooth_radius(d.sigma) > kMediumMaxRad || smooth_radius(d.sigma) < 1)
        throw MediumError(0, "smooth medium: sigma must give a filter radius in [1, 64]");
    Taps T{};
    T.rad = smooth_radius(d.sigma);
    const std::vector<double> g = smooth_taps(d.sigma);
    std::copy(g.begin(), g.end(), T.g);
    // planes of t2 the depth pass reads: reflections of [b - rad, e + rad)
    int64_t L = n0, H = 0;
    for (int64_t p = d.a0_begin - T.rad; p < d.a0_end + T.rad; ++p) {
        const int64_t q = reflect_index(p, n0);
        L = std::min(L, q);
        H = std::max(H, q + 1);
    }
    const int64_t nz = H - L;
    const size_t cnt = static_cast<size_t>(nz * n1 * n2);
    DevBuf<float> t1(cnt), t2(cnt);
    smooth_rows_kernel<<<grid_for(cnt), 256, 0, st>>>(t1.p, L, nz, n1, n2, smooth_salt(d.seed), T);
    MED_CUDA(cudaGetLastError());
    smooth_cols_kernel<<<grid_for(cnt), 256, 0, st>>>(t2.p, t1.p, nz, n1, n2, T);
    MED_CUDA(cudaGetLastError());
    DepthArgs A{};
    A.t2 = t2.p;
    A.L = L;
    A.n0 = n0;
    A.n1 = n1;
    A.n2 = n2;
    A.b = d.a0_begin;
    A.e = d.a0_end;
    A.mode = mode;
    const int64_t total = (d.a0_end - d.a0_begin) * n1 * n2;
    if (mode == 0) {
        DevBuf<unsigned long long> ext(2);
        const unsigned long long init[2] = {~0ull, 0ull};
        MED_CUDA(cudaMemcpyAsync(ext.p, init, sizeof init, cudaMemcpyHostToDevice, st));
        A.ext = ext.p;
        DevBuf<double> sig(1);
        smooth_depth_kernel<<<grid_for(total), 256, 0, st>>>(A, T, sig.p);
        MED_CUDA(cudaGetLastError());
        unsigned long long out[2];
        MED_CUDA(cudaMemcpyAsync(out, ext.p, sizeof out, cudaMemcpyDeviceToHost, st));
        MED_CUDA(cudaStreamSynchronize(st));
        *lo = key_to_double(out[0]);
        *hi = key_to_double(out[1]);
        return;
    }
    if (!(*hi > *lo)) throw MediumError(0, "smooth medium: extrema must satisfy hi > lo");
    const std::vector<double> s = sponge_sigma(d.boundary_width, d.spacing, d.v_min);
    DevBuf<double> sig(s.size());
    MED_CUDA(cudaMemcpyAsync(sig.p, s.data(), sizeof(double) * s.size(), cudaMemcpyHostToDevice, st));
    A.m = m;
    A.eta = eta;
    A.pitch = pitch;
    A.plane = plane;
    A.lo = *lo;
    A.hi = *hi;
    A.v_lo = d.v_lo;
    A.v_hi = d.v_hi;
    A.bw = d.boundary_width;
    smooth_depth_kernel<<<grid_for(total), 256, 0, st>>>(A, T, sig.p);
    MED_CUDA(cudaGetLastError());
    // the temporaries are freed on return: finish with them first
    MED_CUDA(cudaStreamSynchronize(st));
}

} // namespace sfb
