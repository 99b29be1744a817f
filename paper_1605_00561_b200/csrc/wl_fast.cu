// Fast register-tile engine (placeholder until the tuned kernels land).
#include "wl_internal.h"

bool wl_fast_supported(const WlLevel&) { return false; }

cudaError_t wl_launch_fast(const WlLevel&, cudaStream_t) { return cudaErrorNotSupported; }
