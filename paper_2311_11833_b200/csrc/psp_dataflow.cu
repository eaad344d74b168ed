// Fused small-batch factor + forward + backward solve by DATAFLOW (the latency point,
// BASELINE configs[1]: 8 systems): one CTA per perturbed system, its factor image, y and x
// in shared memory, and no level barriers.  Every factor entry, forward row and backward
// row is a task with its contributions in the canonical order (R11):
//   F  entry t = (i, j): v_t <- fma(-l_ip, u_pj, v_t) for p ascending, then (i > j) the
//      division by u_jj, or (i = j) the pivot's status check (R10);
//   Y  row i: y_i <- fma(-l_ip, y_p, y_i), p ascending;
//   X  row i: y_i <- fma(-u_ik, x_k, y_i), k descending, then x_i = y_i / u_ii.
// A contribution waits (acquire loads of per-value ready flags in shared memory) until
// both of its operands are final; a finished task publishes its value with a release
// store.  The host (psp_plan.cpp build_dataflow) sorts the tasks by their finish time in an
// ideal (ASAP) schedule and deals them round-robin to the walkers (one per warp), so every
// walker takes its tasks in a topological order: the unfinished task of least finish time
// can always proceed (no deadlock), and the time is the system's dependency chain rather
// than (levels x barrier).  Same arithmetic as
// the level-scheduled and batch kernels: bitwise equal to them and to the oracle.
// V (batch layout) and X are written at the end for the library's other calls.
#include <climits>
#include <cuda_runtime.h>

#include "psp_dataflow.h"

namespace psp {

namespace {

__device__ __forceinline__ uint32_t df_sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#ifdef PSP_DF_RELAXED
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* f) {
  uint32_t v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(df_sa(f)) : "memory");
  return v;
}
#else
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* f) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(df_sa(f)) : "memory");
  return v;
}
#endif
__device__ __forceinline__ void st_release(uint32_t* f, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(df_sa(f)), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_ready(const uint32_t* f) {
  if (ld_acquire(f) != 0u) return;
  while (ld_acquire(f) == 0u) {
  }
}
__device__ __forceinline__ bool df_pivot_bad(double piv, double tol) {
  return !(fabs(piv) > tol) || !isfinite(piv);
}

__global__ void __launch_bounds__(kDfThreads) dataflow_kernel(const __grid_constant__ DataflowArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int nnz = a.nnz_LU, n = a.n;
  double* v = reinterpret_cast<double*>(dsm);
  double* y = v + nnz;
  double* x = y + n;
  uint32_t* fr = reinterpret_cast<uint32_t*>(x + n);   // factor entries' ready flags
  uint32_t* yr = fr + nnz;
  uint32_t* xr = yr + n;
  uint32_t* pl = reinterpret_cast<uint32_t*>((reinterpret_cast<uintptr_t>(xr + n) + 15) & ~(uintptr_t)15);
  __shared__ int st;
  __shared__ __align__(8) uint64_t pbar;
  const int k = blockIdx.x, tid = threadIdx.x;
  if (tid == 0) {   // the plan arrives by bulk copies while the births are computed
    st = INT_MAX;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(df_sa(&pbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(df_sa(&pbar)),
                 "r"((uint32_t)a.plan_words * 4u) : "memory");
    for (int off = 0; off < a.plan_words; off += 8192) {   // (chunks of 32 KB)
      const int w = min(8192, a.plan_words - off);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              df_sa(pl + off)),
          "l"(a.plan + off), "r"((uint32_t)w * 4u), "r"(df_sa(&pbar))
          : "memory");
    }
  }
  const double e = a.eps[k];
  for (int q = tid; q < nnz; q += kDfThreads) {   // births (a + (eps d) on the diagonal)
    const int sidx = a.birth_src[q], d = a.birth_diag[q];
    const double av = sidx >= 0 ? a.A[sidx] : 0.0;
    v[q] = d >= 0 ? __dadd_rn(av, __dmul_rn(e, a.dperm[d])) : av;
    fr[q] = 0u;
  }
  for (int i = tid; i < n; i += kDfThreads) {
    y[i] = a.b[a.perm[i]];
    yr[i] = 0u;
    xr[i] = 0u;
  }
  const double tol = a.tol_dev ? *a.tol_dev : a.tol_value;
  __syncthreads();
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(df_sa(&pbar))
      : "memory");
  // one walker per warp (lane 0): a spin-wait is then never divergent inside a warp, which
  // would serialise the waiting lanes' loops (measured: 32 walkers per warp ran 2.2x slower
  // than the level-scheduled kernels)
  const int worker = (tid & 31) == 0 ? tid >> 5 : kDfWorkers;
  for (uint32_t w = worker < kDfWorkers ? pl[worker] : 0u, w1 = worker < kDfWorkers ? pl[worker + 1] : 0u;
       w < w1;) {
    const uint32_t h0 = pl[w], h1 = pl[w + 1];
    const uint32_t type = h0 >> 30, cnt = (h0 >> 16) & 0x1fffu;
    const uint32_t* c = pl + w + 2;
    w += 2 + cnt;
    const int t = (int)(h1 & 0xffffu);
    const uint32_t aux = h1 >> 16;
    if (type == 0u) {   // factor entry
      double acc = v[t];
      for (uint32_t q = 0; q < cnt; ++q) {
        const uint32_t lu = c[q];
        const uint32_t l = lu & 0xffffu, u = lu >> 16;
        wait_ready(fr + l);
        wait_ready(fr + u);
        acc = __fma_rn(-v[l], v[u], acc);
      }
      if (aux != 0xffffu) {   // L entry: l = a / u_jj
        wait_ready(fr + aux);
        acc = __ddiv_rn(acc, v[aux]);
      } else if ((h0 >> 29) & 1u) {   // pivot: status (first failing pivot)
        if (df_pivot_bad(acc, tol)) atomicMin(&st, (int)(h0 & 0xffffu) + 1);
      }
      v[t] = acc;
      st_release(fr + t, 1u);
    } else if (type == 1u) {   // forward row
      double acc = y[t];
      for (uint32_t q = 0; q < cnt; ++q) {
        const uint32_t lp = c[q];
        const uint32_t l = lp & 0xffffu, p = lp >> 16;
        wait_ready(fr + l);
        wait_ready(yr + p);
        acc = __fma_rn(-v[l], y[p], acc);
      }
      y[t] = acc;
      st_release(yr + t, 1u);
    } else {   // backward row
      wait_ready(yr + t);
      double acc = y[t];
      for (uint32_t q = 0; q < cnt; ++q) {
        const uint32_t uk = c[q];
        const uint32_t u = uk & 0xffffu, kk = uk >> 16;
        wait_ready(fr + u);
        wait_ready(xr + kk);
        acc = __fma_rn(-v[u], x[kk], acc);
      }
      wait_ready(fr + aux);
      x[t] = __ddiv_rn(acc, v[aux]);
      st_release(xr + t, 1u);
    }
  }
  __syncthreads();
  double* out = a.V + (size_t)(k / a.LS) * nnz * a.LS + (k % a.LS);
  for (int q = tid; q < nnz; q += kDfThreads) out[(size_t)q * a.LS] = v[q];
  double* xo = a.X + (size_t)(k >> 5) * n * 32 + (k & 31);
  for (int i = tid; i < n; i += kDfThreads) xo[(size_t)i * 32] = x[i];
  if (tid == 0) a.status[k] = st == INT_MAX ? 0 : st;
}

}  // namespace

size_t dataflow_smem(int nnz_LU, int n, int plan_words) {
  return sizeof(double) * ((size_t)nnz_LU + 2 * (size_t)n) + sizeof(uint32_t) * ((size_t)nnz_LU + 2 * (size_t)n) +
         sizeof(uint32_t) * (size_t)plan_words + 16;
}

cudaError_t configure_dataflow(size_t smem) {
  return cudaFuncSetAttribute(dataflow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_dataflow(const DataflowArgs& a, int K, size_t smem, cudaStream_t stream) {
  if (K <= 0) return cudaSuccess;
  dataflow_kernel<<<K, kDfThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace psp
