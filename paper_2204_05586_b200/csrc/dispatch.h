// dispatch.h — runtime selection of the compile-time specialised kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ssb {
struct IntervalParams;
using IntervalLaunchFn = cudaError_t (*)(const IntervalParams&, cudaStream_t);
using ExpoLaunchFn = cudaError_t (*)(int64_t, const double*, int, double*, cudaStream_t);
using MagnusLaunchFn = cudaError_t (*)(const IntervalParams&, double*, cudaStream_t);

// One table per (spin, exponentiator, precision) translation unit; index by (method, field).
IntervalLaunchFn interval_table_half_f64(int method, int field);
IntervalLaunchFn interval_table_half_f32(int method, int field);
IntervalLaunchFn interval_table_one_lt_f64(int method, int field);
IntervalLaunchFn interval_table_one_lt_f32(int method, int field);
IntervalLaunchFn interval_table_one_an_f64(int method, int field);
IntervalLaunchFn interval_table_one_an_f32(int method, int field);
IntervalLaunchFn interval_table_one_su3_f64(int method, int field);
IntervalLaunchFn interval_table_one_su3_f32(int method, int field);
ExpoLaunchFn expo_table_half_f64();
ExpoLaunchFn expo_table_half_f32();
ExpoLaunchFn expo_table_one_lt_f64();
ExpoLaunchFn expo_table_one_lt_f32();
ExpoLaunchFn expo_table_one_an_f64();
ExpoLaunchFn expo_table_one_an_f32();
ExpoLaunchFn expo_table_one_su3_f64();
ExpoLaunchFn expo_table_one_su3_f32();
MagnusLaunchFn magnus_table_half_f64(int field);
MagnusLaunchFn magnus_table_half_f32(int field);
MagnusLaunchFn magnus_table_one_lt_f64(int field);
MagnusLaunchFn magnus_table_one_lt_f32(int field);
MagnusLaunchFn magnus_table_one_an_f64(int field);
MagnusLaunchFn magnus_table_one_an_f32(int field);
MagnusLaunchFn magnus_table_one_su3_f64(int field);
MagnusLaunchFn magnus_table_one_su3_f32(int field);
}  // namespace ssb
