// Fused small-batch factor + solve by dataflow (psp_dataflow.cu).  Internal; not part of
// the C ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace psp {

constexpr int kDfThreads = 1024;   // 32 warps
constexpr int kDfWorkers = 32;     // one task walker per warp (lane 0): spin-waits stay warp-uniform

struct DataflowArgs {
  int32_t n = 0, nnz_LU = 0, LS = 32;
  const uint32_t* plan = nullptr;       // psp_plan.h DataflowPlan::words (device)
  int32_t plan_words = 0;
  const int32_t* birth_src = nullptr;   // the cooperative plan's births
  const int32_t* birth_diag = nullptr;
  const int32_t* perm = nullptr;
  const double* A = nullptr;
  const double* eps = nullptr;
  const double* dperm = nullptr;
  const double* b = nullptr;            // one right-hand side, ORIGINAL ordering
  const double* tol_dev = nullptr;
  double tol_value = 0.0;
  double* V = nullptr;                  // factors, batch layout (LS lanes per slab)
  double* X = nullptr;                  // solutions [K/32][1][n][32]
  int32_t* status = nullptr;
};

size_t dataflow_smem(int nnz_LU, int n, int plan_words);
cudaError_t configure_dataflow(size_t smem);
cudaError_t launch_dataflow(const DataflowArgs& a, int K, size_t smem, cudaStream_t stream);

}  // namespace psp
