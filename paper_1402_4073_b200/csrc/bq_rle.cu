// K3/K4: run-length-compressed inputs (placeholder until the device decoder lands).
#include "bq_internal.h"

using namespace bq;

struct bq_rle_query {
    int dummy;
};

extern "C" {
BQ_API int bq_rle_query_create(const bq_rle_span *, int, uint64_t, int, bq_rle_query **out) {
    if (out) *out = nullptr;
    return set_error(BQ_EINPUT, "RLE device path not built yet");
}
BQ_API void bq_rle_query_destroy(bq_rle_query *q) { delete q; }
BQ_API uint64_t bq_rle_query_directory_bytes(const bq_rle_query *) { return 0; }
BQ_API int bq_rle_query_threshold(bq_rle_query *, int, uint64_t *, unsigned long long *, void *) {
    return set_error(BQ_EINPUT, "RLE device path not built yet");
}
BQ_API int bq_rle_query_symmetric(bq_rle_query *, const uint8_t *, uint64_t *, unsigned long long *, void *) {
    return set_error(BQ_EINPUT, "RLE device path not built yet");
}
}
