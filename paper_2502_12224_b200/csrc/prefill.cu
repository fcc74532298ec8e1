// K4 + prefill engine (in progress).
#include "fate_internal.cuh"

extern "C" int fate_ffn_prefill(const float *, int, int, int, const uint8_t *const *, const int32_t *, const float *,
                                const int32_t *, float *, void *) {
  fate::set_error("fate_ffn_prefill: not implemented yet");
  return FATE_EINVAL;
}

extern "C" int fate_engine_prefill(fate_engine *, const double *, const int32_t *, int, float *, fate_prefill_log *,
                                   fate_run_stats *) {
  fate::set_error("fate_engine_prefill: not implemented yet");
  return FATE_EINVAL;
}
