// star.cpp -- placeholder for the 1 draft -> N verifier exchange (filled in next).
#include "abi_internal.h"

using namespace sd;

extern "C" {
sd_status sd_star_unique_ids(int32_t, void*) { return fail(SD_ERR_UNSUPPORTED, "star not built"); }
sd_status sd_star_create(sd_star**, const sd_star_config*, const void*) {
    return fail(SD_ERR_UNSUPPORTED, "star not built");
}
sd_status sd_star_round(sd_star*, const sd_round_desc*, cudaStream_t) {
    return fail(SD_ERR_UNSUPPORTED, "star not built");
}
sd_status sd_star_poll(sd_star*, int32_t*, int32_t*, uint64_t*, int32_t) {
    return fail(SD_ERR_UNSUPPORTED, "star not built");
}
sd_status sd_star_draft_begin(sd_star*, cudaStream_t) { return fail(SD_ERR_UNSUPPORTED, "star not built"); }
sd_status sd_star_draft_end(sd_star*, cudaStream_t) { return fail(SD_ERR_UNSUPPORTED, "star not built"); }
sd_status sd_star_stats(sd_star*, sd_star_stats_t*) { return fail(SD_ERR_UNSUPPORTED, "star not built"); }
sd_status sd_star_destroy(sd_star*) { return fail(SD_ERR_UNSUPPORTED, "star not built"); }
}
