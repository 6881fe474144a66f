// ftc_conv_tc.cu -- placeholder until the tcgen05 engine lands.
#include "ftc_common.cuh"

namespace ftc {
struct TcPlan {};
bool tc_supported(const ftc_conv_desc&) { return false; }
int tc_plan_create(const ftc_conv_desc&, const float*, TcPlan** out, cudaStream_t) {
  *out = nullptr;
  return FTC_CONFIG_ERROR;
}
void tc_plan_destroy(TcPlan* p) { delete p; }
int conv_tc_launch(const TcPlan*, const ConvArgs&, cudaStream_t) { return FTC_CONFIG_ERROR; }
}  // namespace ftc
