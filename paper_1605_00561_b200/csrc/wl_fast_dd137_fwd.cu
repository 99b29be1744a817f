// Instantiation unit of the fast engine: dd137, forward, lifting schemes except Polyphase(*) (reach 3: interpreter).
#include "wl_fast_impl.cuh"

cudaError_t wl_fast_dd137_fwd(int scheme, const WlLevel& L, const wlfast::Plan& p,
                              cudaStream_t s) {
    switch (scheme) {
#define WL_CASE(wi, si, d, P) \
    case si:                  \
        static_assert(P::kReach == wlfast::SchemeConfig<wi, d, si>::KR, "reach"); \
        return wlfast::launch<P, d, wlfast::SchemeConfig<wi, d, si>::R,                    \
                              wlfast::SchemeConfig<wi, d, si>::NW,                   \
                              wlfast::SchemeConfig<wi, d, si>::CPT,                  \
                              wlfast::SchemeConfig<wi, d, si>::NS,                   \
                              wlfast::SchemeConfig<wi, d, si>::XF,                   \
                              wlfast::SchemeConfig<wi, d, si>::MAXB>(L, p, s);
        WL_FAST_FOREACH_2_0(WL_CASE)
#undef WL_CASE
        default:
            return cudaErrorNotSupported;
    }
}
