// Interval-kernel instances: spin/expo/precision = half_f32.
#define SS_SPIN ssb::SPIN_HALF
#define SS_EXPO ssb::EXP_ANALYTIC
#define SS_T float
#define SS_NAME half_f32
#include "interval_instances.inc"
