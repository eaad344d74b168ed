// Pattern-specialised kernels: PTX generated from the symbolic plan, compiled for
// sm_100a with nvJitLink (loaded at run time), cached on disk, loaded with
// cudaLibraryLoadData.  See psp_codegen.cpp.
#pragma once
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace psp {

struct GenInput {
  int32_t n = 0, nnz_L = 0, nnz_LU = 0;
  const std::vector<std::vector<int32_t>>* lcol = nullptr;   // final numbering
  const std::vector<int32_t>* perm = nullptr;                // perm[new] = old
  const std::vector<int32_t>* lofs = nullptr;                // [n+1]
  const std::vector<int32_t>* dofs = nullptr;                // [n+1]
  std::function<int32_t(int32_t, int32_t)> a_index;          // permuted (i,j) -> CSR idx or -1
  int max_regs = 0;                                          // 0: ptxas default (255)
};

// PTX text of the generated kernels (entry points psp_gen_factor, psp_gen_solve).
std::string gen_factor_ptx(const GenInput& g);
std::string gen_solve_ptx(const GenInput& g);

struct GenKernels {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t factor = nullptr;
  cudaKernel_t solve = nullptr;
  std::string cache_file;
  double compile_seconds = 0.0;
  bool from_cache = false;
};

// Compile (or load from the cache) the two kernels.  mode: 1 = cache only, 2 = compile
// when not cached.  load = false only fills the cache (no GPU needed).  Returns false
// with a message in `err` when unavailable.
bool build_gen_kernels(const std::string& factor_ptx, const std::string& solve_ptx, int mode,
                       bool load, GenKernels& out, std::string& err);
void release_gen_kernels(GenKernels& k);

}  // namespace psp
