// integration/sf_cuda_backend.hpp — the reference-side binding a stencilforge
// maintainer adds for CodegenConfig::preset == "cuda" (codegen.hpp:10-19).
//
// This file is written AGAINST the reference's public headers
// (/root/reference/proj/include/sf/*.hpp) and the C ABI of this repository
// (include/sf_b200.h); it is what would live inside stencilforge's op.cpp.
// It is compiled here, unmodified reference alongside, by integration/Makefile
// and exercised on the B200 by tests/test_integration_gpu.py.
//
//   Operator::build()  (op.cpp:94-124, jit_compile at jit.cpp:150-195)
//       -> CudaOperator::CudaOperator: the plan is created from the metadata
//          the reference lowers -- the time function's shape and space order,
//          Options::direction / nt, the h and dt substitutions (Options::subs,
//          acoustic.cpp:168-170), the point counts of the "src" / "rec" sets
//   Operator::apply()  (op.cpp:126-161, CompiledKernel::invoke jit.cpp:104-148)
//       -> CudaOperator::apply: the operator's buffers in KernelSignature
//          order (codegen.cpp:398-409) handed to sf_plan_invoke, status 0 on
//          success, failures raised as the reference's own exception kinds
#pragma once

#include <string>
#include <vector>

#include "sf/op.hpp"

struct sf_plan;

namespace sf_cuda {

class CudaOperator {
  public:
    // `op` is a lowered acoustic or diffusion operator (as acoustic_build /
    // diffusion_operator return it); its grid owns the host buffers
    explicit CudaOperator(sf::Operator& op, int device = 0);
    ~CudaOperator();
    CudaOperator(const CudaOperator&) = delete;
    CudaOperator& operator=(const CudaOperator&) = delete;

    // one call = all nt steps on the GPU, every written buffer back in the
    // grid's host memory on return, like Operator::apply()
    int apply();

    const std::string& kind() const { return kind_; }

  private:
    sf::Operator& op_;
    sf_plan* plan_ = nullptr;
    std::string kind_;
    std::vector<std::string> arg_names_;
};

} // namespace sf_cuda
