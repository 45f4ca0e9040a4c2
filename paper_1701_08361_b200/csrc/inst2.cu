// Line-FFT geometry instantiations, part 2 (see ops.cuh).
#define RTNB_PASS_ONLY
#include "ops.cuh"

namespace rtnb {

void add_ops_2(std::vector<Engine::Ops>& ops, OpsAttrList& attrs) {
  RTNB_INST(12, 16)
  RTNB_INST(16, 16)
  RTNB_INST(16, 20)
}

}  // namespace rtnb
