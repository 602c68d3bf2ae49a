// kernels.h — host-side entry points of the kernels in scan.cu (internal to the library).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include "spinsim_device.cuh"

namespace ssb {
size_t scan_workspace_bytes(int dim, int64_t batch, int64_t k_count);
int64_t chain_min_batch();   // batches from this size take the per-sweep chain kernel (sequential, chunk-invariant)
size_t aggregate_workspace_bytes(int dim, int64_t batch, int64_t k_count);
// op_format: OP_DENSE (U as [batch][k_count][dim][dim] complex128) or OP_SU2 ([batch][k_count][2] complex128, the
// SU(2) element (a, b) of U = [[a, b], [−b*, a*]], acting through D¹ when dim = 3).
cudaError_t launch_scan(int dim, int64_t batch, int64_t k_count, const double* U, const double* psi0, double* states,
                        void* ws, cudaStream_t s, int* launches, double* spin = nullptr, int op_format = OP_DENSE);
// Fused path: coarse scan of the interval kernel's run aggregates run_agg [batch][k_count/seg] (op_format) into the
// run start states phi [batch][k_count/seg + 1][dim], then one chain lane per run of seg ∈ {4, 8, 16, 32} intervals
// (seg | k_count, seg ≤ fused_max_ipt).
cudaError_t launch_fused_scan(int dim, int64_t batch, int64_t k_count, int64_t seg, const double* U,
                              const double* run_agg, const double* psi0, double* phi, double* states, void* ws,
                              cudaStream_t s, int* launches, double* spin = nullptr, int op_format = OP_DENSE);
int fused_max_ipt(int dim, int op_format);
cudaError_t launch_aggregate(int dim, int64_t batch, int64_t k_count, const double* U, double* aggregate, void* ws,
                             cudaStream_t s, int* launches);
cudaError_t launch_compose_carry(int dim, int64_t batch, int part, const double* aggs, const double* psi0,
                                 double* carry, cudaStream_t s);
cudaError_t launch_spin_projection(int dim, int64_t n, const double* states, double* out, cudaStream_t s);
cudaError_t launch_validate(int64_t n_sweep, const double* sweep, int P, int qcol, int64_t n_state,
                            const double* state, int* flag, cudaStream_t s);
}  // namespace ssb
