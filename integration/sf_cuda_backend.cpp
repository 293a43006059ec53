// integration/sf_cuda_backend.cpp — see sf_cuda_backend.hpp. Reference-side
// code: uses only stencilforge's public headers and include/sf_b200.h.
#include "sf_cuda_backend.hpp"

#include <string>

#include "sf/error.hpp"
#include "sf/expr.hpp"
#include "sf/grid.hpp"
#include "sf_b200.h"

namespace sf_cuda {
namespace {

// sf_status -> the reference's exception kinds (error.hpp)
[[noreturn]] void raise(int status, const std::string& where) {
    const std::string msg = where + ": " + sf_last_error();
    switch (status) {
        case SF_ERR_INVALID: throw sf::InvalidShapeError(msg);
        case SF_ERR_CFL: throw sf::CflViolationError(msg);
        case SF_ERR_OUT_OF_DOMAIN: throw sf::OutOfDomainError(msg);
        case SF_ERR_SIGNATURE: throw sf::SignatureMismatchError(msg);
        case SF_ERR_KERNEL: throw sf::KernelFailedError(msg);
        default: throw sf::CompileFailedError(msg);  // no device / CUDA failure
    }
}

// value of the substitution for `sym` in Options::subs (acoustic.cpp:168-170)
double subs_value(const sf::Operator::Options& opt, const sf::Expr& sym) {
    const std::string key = sf::to_string(sym);
    for (const auto& [lhs, rhs] : opt.subs)
        if (sf::to_string(lhs) == key) return rhs.const_value();
    throw sf::UnknownSymbolError("cuda backend: no substitution for " + key);
}

long points_of(const sf::Grid& grid, const char* name, long nt) {
    const sf::GridFunction* gf = grid.find(name);
    if (!gf) throw sf::SignatureMismatchError(std::string("cuda backend: no ") + name + " set");
    return static_cast<long>(gf->numel()) / nt;
}

} // namespace

CudaOperator::CudaOperator(sf::Operator& op, int device) : op_(op) {
    const sf::KernelSignature& sig = op_.signature();  // lowers if needed
    for (const sf::KernelArg& a : sig.args) arg_names_.push_back(a.name);
    const sf::Grid& grid = op_.grid();
    const sf::Operator::Options& opt = op_.options();
    // the acoustic operator of acoustic_build: (u|v, m, eta, src, src_ci,
    // src_w, rec, rec_ci, rec_w) -- golden acoustic_3d.c:3
    const bool acoustic = arg_names_.size() == 9 && arg_names_[1] == "m" && arg_names_[2] == "eta";
    if (!acoustic)
        throw sf::UnloweredConstructError(
            "cuda backend: only the acoustic operator binds here (the generic path is "
            "STENCILFORGE_CC=bin/sf-cuda-cc)");
    kind_ = "acoustic";
    const sf::GridFunction* f = grid.find(arg_names_[0]);
    const std::vector<long> shape = f->space_shape();
    sf_acoustic_desc d{};
    d.ndim = static_cast<int>(shape.size());
    for (int i = 0; i < d.ndim; ++i) d.shape[i] = shape[i];
    d.space_order = f->space_order();
    d.forward = opt.direction == sf::Direction::forward ? 1 : 0;
    d.nt = opt.nt;
    d.dt = subs_value(opt, sf::symbols::s());
    d.spacing = subs_value(opt, sf::symbols::h());
    d.n_src = points_of(grid, "src", opt.nt);
    d.n_rec = points_of(grid, "rec", opt.nt);
    if (int rc = sf_acoustic_plan_create(&d, device, &plan_)) raise(rc, "sf_acoustic_plan_create");
}

CudaOperator::~CudaOperator() {
    if (plan_) sf_plan_destroy(plan_);
}

int CudaOperator::apply() {
    sf::Grid& grid = op_.grid();
    std::vector<void*> args;  // KernelSignature order, as CompiledKernel::invoke
    for (const std::string& n : arg_names_) args.push_back(grid.find(n)->data());
    const int status = sf_plan_invoke(plan_, args.data(), static_cast<int>(args.size()));
    if (status != 0) raise(status, "sf_plan_invoke");
    return status;
}

} // namespace sf_cuda
