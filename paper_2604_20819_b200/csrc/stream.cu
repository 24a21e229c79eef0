// Streamed forward (Q/K/V in pinned host memory): placeholder until the staging executor lands.
#include <cuda_runtime.h>

#include "cqs_internal.h"

namespace cqs {
cqs_status forward_streamed(const cqs_plan_t*, const void*, const void*, const void*, void*,
                            const int64_t*, float*, float, uint8_t*, uint8_t*, cudaStream_t,
                            cqs_stats*) {
  return fail(CQS_E_UNSUPPORTED, "streamed (pinned host) Q/K/V not built yet");
}
}  // namespace cqs
