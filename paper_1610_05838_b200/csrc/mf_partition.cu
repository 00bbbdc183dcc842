// mf_partition.cu -- multi-GPU block partition with Q rotation (§4.1).  [stub]
#include "mf_ctx.h"

int mf_ctx::epoch_partitioned(mf_epoch_stats *) { return fail(MF_EINVAL, "partitioned schedule not built yet"); }
int mf_ctx::rmse_partitioned(int64_t, double *) { return fail(MF_EINVAL, "partitioned schedule not built yet"); }
int mf_ctx::gather_q() { return MF_OK; }
void mf_ctx::release_partition() {}
extern "C" int mf_nccl_unique_id(void *) { return MF_ENCCL; }
extern "C" int mf_attach_nccl(mf_ctx *, const void *, int, int) { return MF_ENCCL; }
extern "C" int mf_segment(int64_t extent, int32_t parts, int32_t index, int64_t *b, int64_t *e) {
    if (extent < 0 || parts <= 0 || index < 0 || index >= parts || !b || !e) return MF_EINVAL;
    *b = extent * index / parts;
    *e = extent * (index + 1) / parts;
    return MF_OK;
}
extern "C" int mf_round_segment(uint64_t, int32_t, int32_t, int32_t, int32_t, int32_t *) { return MF_EINVAL; }
