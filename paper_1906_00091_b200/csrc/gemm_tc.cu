// tcgen05 3xTF32 GEMMs — placeholder until the tensor-core kernels land;
// every predicate declines so the SIMT path runs.
#include "gemm_tc.cuh"

namespace dlrm {

bool tc_linear_fwd_ok(const float*, int64_t, const float*, int64_t,
                      const float*, int64_t, int64_t, int64_t, int64_t,
                      int64_t) {
  return false;
}
int tc_linear_fwd(const float*, int64_t, const float*, int64_t, const float*,
                  float*, int64_t, int64_t, int64_t, int64_t, int64_t, int,
                  cudaStream_t) {
  set_error("tcgen05 linear_fwd not built");
  return 1;
}
bool tc_linear_bwd_data_ok(const float*, int64_t, const float*, int64_t,
                           const float*, int64_t, int64_t, int64_t, int64_t) {
  return false;
}
int tc_linear_bwd_data(const float*, int64_t, const float*, int64_t,
                       const float*, int64_t, float*, int64_t, int64_t,
                       int64_t, int64_t, cudaStream_t) {
  set_error("tcgen05 linear_bwd_data not built");
  return 1;
}
bool tc_linear_bwd_weight_ok(const float*, int64_t, const float*, int64_t,
                             int64_t, int64_t, int64_t) {
  return false;
}
size_t tc_linear_bwd_weight_ws_floats(int64_t, int64_t, int64_t) { return 0; }
int tc_linear_bwd_weight(const float*, int64_t, const float*, int64_t, int64_t,
                         int64_t, int64_t, float*, int64_t, float*, int64_t,
                         float, const int32_t*, float*, cudaStream_t) {
  set_error("tcgen05 linear_bwd_weight not built");
  return 1;
}

}  // namespace dlrm
