// Temporary: PCDM and Newton-CG drivers land in pcdm.cu / ncg.cu.
#include "solvers.hpp"

namespace l1b {
void run_pcdm(l1b_problem*, const l1b_solver_cfg*, l1b_sample*, uint64_t, l1b_summary*, double*,
              double*) {
  throw Unsupported("pcdm: not built yet");
}
void run_newton_cg(l1b_problem*, const l1b_solver_cfg*, l1b_sample*, uint64_t, l1b_summary*,
                   double*, double*) {
  throw Unsupported("newton_cg: not built yet");
}
}  // namespace l1b
