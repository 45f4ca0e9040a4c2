// Line-FFT geometry instantiations, part 2 (see ops.cuh).
#define RTNB_PASS_ONLY
#include "ops.cuh"

namespace rtnb {

void add_ops_2(std::vector<Engine::Ops>& ops, OpsAttrList& attrs) {
  RTNB_INST(12, 16)
  ops.push_back(Inst<16, 16>::make());
  Inst<16, 16>::add_cluster<8>(ops.back());
  attrs.push_back({16 * 16, &Inst<16, 16>::set_attrs});
  RTNB_INST(20, 16)  // k_rows2 at G = 320 (C2): faster than 16 x 20 (ops_for merges)
  RTNB_INST(16, 20)
}

}  // namespace rtnb
