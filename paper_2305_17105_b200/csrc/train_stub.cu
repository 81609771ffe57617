// placeholder until train.cu lands
#include "common.cuh"
extern "C" {
struct ntc_trainer { int dummy; };
ntc_status ntc_trainer_create(const ntc_desc*, ntc_trainer** out) { *out = nullptr; return NTC_ERR_UNSUPPORTED; }
void ntc_trainer_destroy(ntc_trainer*) {}
ntc_status ntc_train_step(ntc_trainer*, const ntc_desc*, const ntc_train_buffers*, const ntc_batch*,
                          const ntc_train_hparams*, float*, int32_t*, uint32_t, ntc_stream) { return NTC_ERR_UNSUPPORTED; }
int32_t ntc_train_footprint(const ntc_desc*, const ntc_batch*, int32_t*) { return 0; }
}
