// hlm_crew.cu -- CREW variant (local_max_par.hpp:258-338): placeholder until the segmented-max
// kernels land; fails loudly instead of falling back.
#include "hlm_engine.h"

namespace hlmb {

int match_crew(Graph*, const hlm_b200_stream*, const hlm_b200_config*, hlm_b200_result*) {
  set_error("crew variant not built yet");
  return HLM_B200_ERR_UNSUPPORTED;
}

void crew_release(Graph*) {}

}  // namespace hlmb
