// integration/backend_check.cpp — drives the reference-side binding
// (sf_cuda_backend.hpp) the way a stencilforge user would: build the acoustic
// operator with the reference's own acoustic_build (acoustic.cpp:128-200),
// run one copy through the reference's JIT'd C (Operator::apply) and an
// identical copy through sf_cuda::CudaOperator on the B200, then require
// every buffer of the two grids to be bitwise equal. Prints one JSON line per
// case; exit status 0 when all match.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "sf/acoustic.hpp"
#include "sf_cuda_backend.hpp"

namespace {

struct Case {
    std::vector<long> shape;
    int order;
    bool forward;
    long nt;
};

bool run_case(const Case& c) {
    sf::AcousticModel model;
    model.shape = c.shape;
    model.boundary_width = 6;
    model.spacing = 10.0;
    model.nt = c.nt;
    model.space_order = c.order;
    sf::AcousticSetup a = sf::acoustic_build(model, c.forward);
    sf::AcousticSetup b = sf::acoustic_build(model, c.forward);
    if (!c.forward) {  // a seeded residual at the receivers (both copies)
        std::mt19937_64 rng(11);
        std::normal_distribution<double> n01(0.0, 1.0);
        for (long t = 0; t < c.nt; ++t)
            for (long p = 0; p < a.rec->num_points(); ++p) {
                const double v = n01(rng);
                a.rec->set_series(t, p, v);
                b.rec->set_series(t, p, v);
            }
    }
    a.op->apply();  // the reference: JIT'd C99/OpenMP on the host
    sf_cuda::CudaOperator cuda(*b.op);
    cuda.apply();   // the binding: the B200 plan through sf_plan_invoke
    long compared = 0, mismatched = 0;
    std::string bad;
    for (const auto& gf : a.grid->functions()) {
        const sf::GridFunction* other = b.grid->find(gf->name());
        if (!other || other->bytes() != gf->bytes()) {
            ++mismatched;
            bad += gf->name() + "(layout) ";
            continue;
        }
        ++compared;
        if (std::memcmp(gf->data(), other->data(), gf->bytes()) != 0) {
            ++mismatched;
            bad += gf->name() + " ";
        }
    }
    double peak = 0.0;
    const float* u = static_cast<const float*>(b.field->data());
    for (size_t i = 0; i < b.field->numel(); ++i) peak = std::max(peak, (double)std::fabs(u[i]));
    std::string shape;
    for (long e : c.shape) shape += (shape.empty() ? "" : "x") + std::to_string(e);
    std::printf("{\"case\": \"%s order %d %s nt %ld\", \"kind\": \"%s\", \"buffers\": %ld, "
                "\"mismatched\": %ld, \"bad\": \"%s\", \"field_peak\": %.6g}\n",
                shape.c_str(), c.order, c.forward ? "forward" : "adjoint", c.nt,
                cuda.kind().c_str(), compared, mismatched, bad.c_str(), peak);
    std::fflush(stdout);
    return mismatched == 0 && compared >= 9 && peak > 0.0;
}

} // namespace

int main() {
    const Case cases[] = {
        {{40, 36, 44}, 4, true, 30},  {{40, 36, 44}, 8, true, 30},
        {{44, 40, 48}, 16, true, 20}, {{40, 36, 44}, 8, false, 30},
        {{80, 70}, 8, true, 60},      {{80, 70}, 4, false, 60},
    };
    int failures = 0;
    for (const Case& c : cases) {
        try {
            if (!run_case(c)) ++failures;
        } catch (const std::exception& e) {
            std::printf("{\"error\": \"%s\"}\n", e.what());
            ++failures;
        }
    }
    return failures == 0 ? 0 : 1;
}
