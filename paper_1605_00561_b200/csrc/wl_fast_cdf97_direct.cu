// Instantiation unit of the fast engine: cdf97, direct-load variant (no TMA;
// wlfast::launch_direct), both directions, all lifting schemes.
#include "wl_fast_impl.cuh"

cudaError_t wl_fast_cdf97_direct(int scheme, const WlLevel& L, const wlfast::Plan& p,
                               cudaStream_t s) {
#define WL_CASE(wi, si, d, P)                                                               \
    case si:                                                                                \
        return wlfast::launch_direct<P, d, wlfast::DirectConfigOf<wi, d, si>::R,              \
                                     wlfast::DirectConfigOf<wi, d, si>::NW,                   \
                                     wlfast::DirectConfigOf<wi, d, si>::CPT,                  \
                                     wlfast::DirectConfigOf<wi, d, si>::NS,                   \
                                     wlfast::DirectConfigOf<wi, d, si>::XF,                   \
                                     wlfast::DirectConfigOf<wi, d, si>::MAXB>(L, p, s);
    if (L.direction == 0) {
        switch (scheme) {
            WL_FAST_FOREACH_1_0(WL_CASE)
            default:
                return cudaErrorNotSupported;
        }
    }
    switch (scheme) {
        WL_FAST_FOREACH_1_1(WL_CASE)
        default:
            return cudaErrorNotSupported;
    }
#undef WL_CASE
}
