// mf_wavefront.cu -- wavefront-update schedule (§3.2.3).  [stub: filled in next]
#include "mf_ctx.h"

int mf_ctx::build_wavefront() { return fail(MF_EINVAL, "wavefront schedule not built yet"); }
int mf_ctx::run_wavefront(const mf::ShapeId &, const mf::UpdateArgs &, int *, int *) {
    return fail(MF_EINVAL, "wavefront schedule not built yet");
}
void mf_ctx::release_wavefront() {}
extern "C" int mf_wavefront_trace(mf_ctx *ctx, int64_t *, int64_t, int64_t *count) {
    if (!ctx || !count) return MF_EINVAL;
    *count = 0;
    return MF_OK;
}
