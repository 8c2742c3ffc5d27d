// tcgen05 (5th-generation tensor core) version of the training tile: placeholder
// until the UMMA kernel lands; the runtime falls back to nothing — callers
// select WG_MLP_EXACT explicitly when this reports unavailable.
#include "wg_train.cuh"

namespace wg {
bool tc_grad_available() { return false; }
cudaError_t launch_grad_tc(const TrainArgs&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace wg
