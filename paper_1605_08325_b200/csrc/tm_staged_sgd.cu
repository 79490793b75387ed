// sm_100a staged exchange with the momentum-SGD step of tm_bsp_step fused into
// the pre-cast (ExchangeArgs::sgd): the SGD = true instantiations
// of the kernels in tm_staged.cuh, in their own translation unit.
#include "tm_staged.cuh"

namespace tmx {

const void* pick_exchange_sgd(int k, bool w16, bool sys, int fl) {
  return pick_exchange<true>(k, w16, sys, fl);
}

}  // namespace tmx
