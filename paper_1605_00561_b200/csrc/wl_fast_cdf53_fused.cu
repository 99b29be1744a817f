// Instantiation unit of the fast engine: cdf53, two fused forward pyramid
// levels (wlfast::launch_fused), all lifting schemes.
#include "wl_fast_impl.cuh"

cudaError_t wl_fast_cdf53_fwd_fused(int scheme, const WlLevel& L0, const wlfast::Plan& p0,
                                   const WlLevel& L1, const wlfast::Plan& p1, unsigned* ctr,
                                   cudaStream_t s) {
    switch (scheme) {
#define WL_CASE(wi, si, d, P)                                                               \
    case si:                                                                                \
        return wlfast::launch_fused<P, d, wlfast::SchemeConfig<wi, d, si>::R,               \
                                    wlfast::SchemeConfig<wi, d, si>::NW,                    \
                                    wlfast::SchemeConfig<wi, d, si>::CPT,                   \
                                    wlfast::SchemeConfig<wi, d, si>::NS,                    \
                                    wlfast::SchemeConfig<wi, d, si>::XF,                    \
                                    wlfast::SchemeConfig<wi, d, si>::MAXB>(L0, p0, L1, p1,  \
                                                                          ctr, s);
        WL_FAST_FOREACH_0_0(WL_CASE)
#undef WL_CASE
        default:
            return cudaErrorNotSupported;
    }
}
