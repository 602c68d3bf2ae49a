// Interval-kernel instances: spin/expo/precision = one_an_f32.
#define SS_SPIN ssb::SPIN_ONE
#define SS_EXPO ssb::EXP_ANALYTIC
#define SS_T float
#define SS_NAME one_an_f32
#include "interval_instances.inc"
