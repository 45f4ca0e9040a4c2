// Line-FFT geometry instantiations, part 1 (see ops.cuh).
#define RTNB_PASS_ONLY
#include "ops.cuh"

namespace rtnb {

void add_ops_1(std::vector<Engine::Ops>& ops, OpsAttrList& attrs) {
  RTNB_INST(8, 9)
  RTNB_INST(8, 12)
  ops.push_back(Inst<8, 16>::make());  // G = 128 (C1): also one cluster per channel
  Inst<8, 16>::add_cluster<8>(ops.back());
  attrs.push_back({8 * 16, &Inst<8, 16>::set_attrs});
  RTNB_INST(10, 16)
}

}  // namespace rtnb
