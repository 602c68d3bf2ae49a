// Interval-kernel instances: spin/expo/precision = one_su3_f32 (general spin-one, readings R19/R20).
#define SS_SPIN ssb::SPIN_ONE
#define SS_EXPO ssb::EXP_LIE_TROTTER_SU3
#define SS_T float
#define SS_NAME one_su3_f32
#define SS_SU3 1
#include "interval_instances.inc"
