// user_field.h — run-time compiled user field functions (internal to the library).
#pragma once
#include <string>

#include <cuda_runtime.h>

namespace ssb {
struct IntervalParams;
struct UserKernel {
  void* module = nullptr;     // CUmodule
  void* function = nullptr;   // CUfunction (interval kernel)
  void* magnus = nullptr;     // CUfunction (Magnus diagnostic)
};
// spin: 1 (half) / 2 (one); expo, method as ss_expo / ss_integration; returns 0 or < 0 with *err set.
// out == nullptr: compile only (no device, no module load).
int build_user_kernel(int spin, int expo, int method, int fp32, const char* field_src, int n_params, UserKernel* out,
                      std::string* err);
cudaError_t launch_user(const UserKernel& k, const IntervalParams& prm, cudaStream_t stream);
cudaError_t launch_user_magnus(const UserKernel& k, const IntervalParams& prm, double* out, cudaStream_t stream);
void destroy_user_kernel(UserKernel* k);
}  // namespace ssb
