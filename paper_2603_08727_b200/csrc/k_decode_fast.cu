// k_decode_fast.cu — tensor-core decode attention for FRAG-layout caches (placeholder
// until the mma.sync kernel lands; the generic kernel serves every cache meanwhile).
#include "kernels.h"

namespace arkv {
int launch_decode_fast(const DecodeArgs&, int, cudaStream_t, cudaEvent_t, cudaEvent_t) { return -1; }
}  // namespace arkv
