// Line-FFT geometry instantiations, part 0 (see ops.cuh).
#define RTNB_PASS_ONLY
#include "ops.cuh"

namespace rtnb {

void add_ops_0(std::vector<Engine::Ops>& ops, OpsAttrList& attrs) {
  RTNB_INST(4, 4)
  RTNB_INST(4, 6)
  RTNB_INST(4, 8)
  RTNB_INST(6, 8)
  RTNB_INST(8, 8)
}

}  // namespace rtnb
