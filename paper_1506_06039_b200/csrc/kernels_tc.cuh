// kernels_tc.cuh -- tensor-core (tcgen05, kind::i8) exact coarse search.
// Placeholder interface; the implementation lands with the TC path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace moco {

struct TcPlan {
  bool ready = false;
  bool tpl_ready = false;
};

inline bool tc_supported(int dtype, int bits, int levels, int w, int mc, int nc) {
  (void)dtype; (void)bits; (void)levels; (void)w; (void)mc; (void)nc;
  return false;
}
inline bool tc_auto_prefers(int w) { (void)w; return false; }
inline int tc_init(TcPlan *, int, int, int, int64_t) { return -1; }
inline int tc_set_template(TcPlan *, const uint16_t *, int, cudaStream_t) { return -1; }
inline int tc_coarse(TcPlan *, const uint16_t *, int64_t, int, int, const unsigned long long *,
                     double, int32_t *, double *, uint8_t *, cudaStream_t, int64_t *) {
  return -1;
}
inline void tc_free(TcPlan *) {}

}  // namespace moco
