// oracle/ref_driver.cpp — C-ABI harness over the UNMODIFIED reference library
// (stencilforge, /root/reference/proj) so Python tests, the golden-fixture
// generator and bench.py's CPU arm can drive it through ctypes.
//
// TEST INFRASTRUCTURE: this file is the checker, never the product. It only
// calls the reference's public API:
//   acoustic_build            acoustic.cpp:128-206   (AcousticModel, acoustic.hpp:17-42)
//   diffusion build/run       diffusion.cpp:86-140
//   Operator::apply/source/nest  op.cpp:94-161
//   interpolation_weights     sparse.cpp:11-41
//   GridFunction data access  grid.hpp:32-98
// Buffers are exchanged by GridFunction name in the reference's own dense
// row-major layout (slot slowest, grid.cpp:89-101).
#include <omp.h>

#include <random>

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "sf/acoustic.hpp"
#include "sf/diffusion.hpp"
#include "sf/error.hpp"
#include "sf/sparse.hpp"

using namespace sf;

namespace {

thread_local std::string g_err;
thread_local std::string g_text;
thread_local BlockingPlan g_blocking; // applied to the next build (opt.hpp:10-15)

struct Handle {
    std::unique_ptr<Grid> grid_owner; // diffusion
    AcousticSetup acoustic;           // acoustic (owns its grid)
    DiffusionBuild diffusion;
    Operator* op = nullptr;
    Grid* grid = nullptr;
    double dt = 0.0;
};

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const CflViolationError& e) {
        g_err = std::string("CflViolationError: ") + e.what();
        return 2;
    } catch (const OutOfDomainError& e) {
        g_err = std::string("OutOfDomainError: ") + e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

std::vector<std::vector<double>> unpack(int n, int dims, const double* c) {
    std::vector<std::vector<double>> out;
    for (int p = 0; p < n; ++p)
        out.emplace_back(c + static_cast<size_t>(p) * dims,
                         c + static_cast<size_t>(p + 1) * dims);
    return out;
}

} // namespace

extern "C" {

const char* sfref_last_error() { return g_err.c_str(); }

void sfref_set_threads(int n) { omp_set_num_threads(n); }

// Blocking plan for the next acoustic/diffusion build: sizes for the spatial
// dimensions "x", "y", "z" (grid.cpp:47); size 0 leaves a dimension unblocked.
void sfref_set_blocking(int n, const long* sizes) {
    static const char* names[3] = {"x", "y", "z"};
    g_blocking = BlockingPlan{};
    for (int d = 0; d < n && d < 3; ++d)
        if (sizes[d] > 0) g_blocking.block[names[d]] = sizes[d];
}
int sfref_max_threads() { return omp_get_max_threads(); }

// Acoustic forward (forward != 0) or adjoint operator, built but not run.
// dt <= 0 derives stable_dt (acoustic.hpp:31-33). Coordinates are metres,
// row-major [n][ndim]; n == 0 selects the model's defaults.
void* sfref_acoustic_build(int ndim, const long* shape, int boundary_width,
                           double spacing, long nt, double dt, int order,
                           double f0, double v_top, double v_bottom,
                           int nsrc, const double* src_coords, int nrec,
                           const double* rec_coords, int forward) {
    Handle* h = new Handle;
    int rc = guard([&] {
        AcousticModel m;
        m.shape.assign(shape, shape + ndim);
        m.boundary_width = boundary_width;
        m.spacing = spacing;
        m.nt = nt;
        m.dt = dt;
        m.space_order = order;
        m.f0 = f0;
        m.v_top = v_top;
        m.v_bottom = v_bottom;
        if (nsrc > 0) m.src_coords = unpack(nsrc, ndim, src_coords);
        if (nrec > 0) m.rec_coords = unpack(nrec, ndim, rec_coords);
        m.blocking = g_blocking;
        h->acoustic = acoustic_build(m, forward != 0);
        h->op = h->acoustic.op.get();
        h->grid = h->acoustic.grid.get();
        h->dt = h->acoustic.dt;
    });
    if (rc != 0) {
        delete h;
        return nullptr;
    }
    return h;
}

double sfref_acoustic_stable_dt(int ndim, const long* shape, double spacing,
                                int order, double v_top, double v_bottom) {
    AcousticModel m;
    m.shape.assign(shape, shape + ndim);
    m.spacing = spacing;
    m.space_order = order;
    m.v_top = v_top;
    m.v_bottom = v_bottom;
    return m.stable_dt();
}

double sfref_ricker(double f0, double t, double t0) {
    return ricker_wavelet(f0, t, t0);
}

// Diffusion operator (diffusion.cpp:86-113) with rational alpha / dx.
void* sfref_diffusion_build(long nx, long ny, long alpha_num, long alpha_den,
                            long dx_num, long dx_den, long nt, int order) {
    Handle* h = new Handle;
    int rc = guard([&] {
        DiffusionConfig c;
        c.nx = nx;
        c.ny = ny;
        c.alpha = Rational(alpha_num, alpha_den);
        c.dx = c.dy = Rational(dx_num, dx_den);
        c.nt = nt;
        c.order = order;
        c.blocking = g_blocking;
        h->dt = c.dt().to_double();
        h->diffusion = make_diffusion_operator(c);
        h->op = h->diffusion.op.get();
        h->grid = h->diffusion.grid.get();
    });
    if (rc != 0) {
        delete h;
        return nullptr;
    }
    return h;
}

void sfref_free(void* hp) { delete static_cast<Handle*>(hp); }

double sfref_dt(void* hp) { return static_cast<Handle*>(hp)->dt; }

long sfref_buffer_bytes(void* hp, const char* name) {
    Handle* h = static_cast<Handle*>(hp);
    GridFunction* gf = h->grid->find(name);
    return gf ? static_cast<long>(gf->bytes()) : -1;
}

int sfref_get(void* hp, const char* name, void* out, long bytes) {
    Handle* h = static_cast<Handle*>(hp);
    GridFunction* gf = h->grid->find(name);
    if (!gf || static_cast<long>(gf->bytes()) != bytes) {
        g_err = std::string("no buffer / size mismatch: ") + name;
        return 1;
    }
    std::memcpy(out, gf->data(), gf->bytes());
    return 0;
}

int sfref_set(void* hp, const char* name, const void* in, long bytes) {
    Handle* h = static_cast<Handle*>(hp);
    GridFunction* gf = h->grid->find(name);
    if (!gf || static_cast<long>(gf->bytes()) != bytes) {
        g_err = std::string("no buffer / size mismatch: ") + name;
        return 1;
    }
    std::memcpy(gf->data(), in, gf->bytes());
    return 0;
}

// JIT-compile (gcc, jit.cpp:150-195) without running.
int sfref_build(void* hp) {
    Handle* h = static_cast<Handle*>(hp);
    return guard([&] { h->op->build(); });
}

// Operator::apply(): all nt steps of the generated C/OpenMP kernel.
int sfref_apply(void* hp) {
    Handle* h = static_cast<Handle*>(hp);
    return guard([&] { h->op->apply(); });
}

const char* sfref_source(void* hp) {
    Handle* h = static_cast<Handle*>(hp);
    int rc = guard([&] { g_text = h->op->source(); });
    return rc == 0 ? g_text.c_str() : nullptr;
}

// Lowered, folded, CSE'd loop nest with full-precision constants
// (ir.cpp:400-457 printer).
const char* sfref_nest(void* hp) {
    Handle* h = static_cast<Handle*>(hp);
    int rc = guard([&] { g_text = to_string(h->op->nest()); });
    return rc == 0 ? g_text.c_str() : nullptr;
}

// interpolation_weights (sparse.cpp:11-41) for one point.
int sfref_interp_weights(int ndim, const double* coord, double spacing,
                         const long* extents, long* cell_out,
                         double* weights_out) {
    return guard([&] {
        InterpWeights w = interpolation_weights(
            std::span<const double>(coord, ndim), spacing,
            std::span<const long>(extents, ndim));
        for (int i = 0; i < ndim; ++i) cell_out[i] = w.cell[i];
        for (size_t k = 0; k < w.weights.size(); ++k)
            weights_out[k] = w.weights[k];
    });
}

} // extern "C"

extern "C" {
// std::mt19937_64(seed) + std::uniform_real_distribution<double>(lo, hi),
// the draw sequence adjoint_test uses (acoustic.cpp:230-235).
void sfref_mt_uniform(unsigned seed, long n, double lo, double hi, double* out) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(lo, hi);
    for (long i = 0; i < n; ++i) out[i] = dist(rng);
}

// adjoint_test (acoustic.cpp:223-237) through the reference: fills the
// four products, returns 0.
int sfref_adjoint_test(int ndim, const long* shape, int boundary_width, double spacing,
                       long nt, int order, unsigned seed, double* out4) {
    return guard([&] {
        AcousticModel m;
        m.shape.assign(shape, shape + ndim);
        m.boundary_width = boundary_width;
        m.spacing = spacing;
        m.nt = nt;
        m.space_order = order;
        AdjointTestResult r = adjoint_test(m, seed);
        out4[0] = r.forward_product;
        out4[1] = r.adjoint_product;
        out4[2] = r.difference;
        out4[3] = r.ratio;
    });
}
}

extern "C" {
// save_buffer / load_buffer (grid.cpp:213-254) on a named GridFunction.
int sfref_save_buffer(void* hp, const char* name, const char* path) {
    Handle* h = static_cast<Handle*>(hp);
    return guard([&] { save_buffer(*h->grid->find(name), path); });
}
int sfref_load_buffer(void* hp, const char* name, const char* path) {
    Handle* h = static_cast<Handle*>(hp);
    return guard([&] { load_buffer(*h->grid->find(name), path); });
}
// dump_csv (grid.cpp:256-273) and save_series_text (sparse.cpp:215-227)
int sfref_dump_csv(void* hp, const char* name, const char* path, long slot) {
    Handle* h = static_cast<Handle*>(hp);
    return guard([&] { dump_csv(*h->grid->find(name), path, slot); });
}
int sfref_save_series_text(void* hp, const char* name, const char* path) {
    Handle* h = static_cast<Handle*>(hp);
    return guard([&] { save_series_text(*h->grid->find(name), path); });
}
// load_series_column (sparse.cpp:205-213): returns the count, fills up to cap
long sfref_load_series_column(const char* path, double* out, long cap) {
    long n = -1;
    guard([&] {
        std::vector<double> v = load_series_column(path);
        n = static_cast<long>(v.size());
        for (long i = 0; i < n && i < cap; ++i) out[i] = v[i];
    });
    return n;
}
}
