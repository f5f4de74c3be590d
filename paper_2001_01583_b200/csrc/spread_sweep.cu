// spread_sweep.cu -- placeholder until the column-sweep kernel lands.
#include "spread_common.cuh"

namespace hpnfft {

bool sweep_supported(const Plan* p) {
  (void)p;
  return false;
}

int spread_sweep(Plan* p, const double* f) {
  (void)f;
  set_error("sweep spread not built");
  return HPNFFT_E_UNSUPPORTED;
}

}  // namespace hpnfft
