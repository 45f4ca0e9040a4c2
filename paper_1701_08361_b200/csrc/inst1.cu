// Line-FFT geometry instantiations, part 1 (see ops.cuh).
#define RTNB_PASS_ONLY
#include "ops.cuh"

namespace rtnb {

void add_ops_1(std::vector<Engine::Ops>& ops, OpsAttrList& attrs) {
  RTNB_INST(8, 9)
  RTNB_INST(8, 12)
  RTNB_INST(8, 16)
  RTNB_INST(10, 16)
}

}  // namespace rtnb
