// k_disc_tc.cu -- bf16 discriminator on the 5th-generation tensor cores
// (tcgen05 + TMEM).  Placeholder until the fused kernel lands: the BF16
// precision reports UNSUPPORTED at create time.
#include "ctx.h"

namespace sagips {

bool tc_disc_supported(const sagips_config*) { return false; }
sagips_status tc_disc_init(sagips_ctx*) { return SAGIPS_ERR_UNSUPPORTED; }
void tc_disc_destroy(sagips_ctx*) {}
void tc_disc_step(sagips_ctx*, cudaStream_t) {}
void tc_gen_loss(sagips_ctx*, cudaStream_t) {}

}  // namespace sagips
