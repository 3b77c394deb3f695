// reg_v3_fast.cu -- v3 launches, FAST arithmetic (see reg_v3.inc).
#include "reg_v3.inc"

namespace sconv_cu {
namespace host {
int launch_ws_fast(sconv_cu_ctx* ctx, int which, int P, const WsArgs& a) {
  return launch_ws<true>(ctx, which, P, a);
}
}  // namespace host
}  // namespace sconv_cu
