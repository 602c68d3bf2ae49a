// Interval-kernel instances: spin/expo/precision = half_f64.
#define SS_SPIN ssb::SPIN_HALF
#define SS_EXPO ssb::EXP_ANALYTIC
#define SS_T double
#define SS_NAME half_f64
#include "interval_instances.inc"
