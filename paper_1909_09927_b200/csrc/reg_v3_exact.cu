// reg_v3_exact.cu -- v3 launches, EXACT arithmetic (see reg_v3.inc).
#include "reg_v3.inc"

namespace sconv_cu {
namespace host {
int launch_ws_exact(sconv_cu_ctx* ctx, int which, int P, const WsArgs& a) {
  return launch_ws<false>(ctx, which, P, a);
}
}  // namespace host
}  // namespace sconv_cu
