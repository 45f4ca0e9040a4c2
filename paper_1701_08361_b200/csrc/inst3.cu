// Line-FFT geometry instantiations, part 3 (see ops.cuh).
#define RTNB_PASS_ONLY
#include "ops.cuh"

namespace rtnb {

void add_ops_3(std::vector<Engine::Ops>& ops, OpsAttrList& attrs) {
  RTNB_INST(16, 24)
  RTNB_INST(24, 16)  // measured faster at G = 384 (C5): the later registration wins
  RTNB_INST(16, 32)
}

}  // namespace rtnb
