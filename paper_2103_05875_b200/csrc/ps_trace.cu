// Stages (1)+(2): probe ray tracing + DDGI blend.  (bring-up placeholder)
#include "ps_common.cuh"

using namespace ps;

extern "C" {
int ps_bvh_build(const double *, int64_t, int, ps_bvh_sizes *, float *, float *) {
    PS_ABI_BEGIN
    fail(PS_ERR_VALUE, "ps_bvh_build: not available in this build");
    PS_ABI_END
}
int ps_blend_weights(const float *, int32_t, const float *, float, float *, float *, float *,
                     void *) {
    PS_ABI_BEGIN
    fail(PS_ERR_VALUE, "ps_blend_weights: not available in this build");
    PS_ABI_END
}
int ps_trace_blend(const ps_trace_params *, void *) {
    PS_ABI_BEGIN
    fail(PS_ERR_VALUE, "ps_trace_blend: not available in this build");
    PS_ABI_END
}
}
