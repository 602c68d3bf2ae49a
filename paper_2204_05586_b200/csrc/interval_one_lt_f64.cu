// Interval-kernel instances: spin/expo/precision = one_lt_f64.
#define SS_SPIN ssb::SPIN_ONE
#define SS_EXPO ssb::EXP_LIE_TROTTER
#define SS_T double
#define SS_NAME one_lt_f64
#include "interval_instances.inc"
