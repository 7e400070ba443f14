// lv_encoder.cuh — internal interface of the passage encoder (lv_encoder.cu).
#pragma once
#include "lv_common.cuh"

namespace lv {

int encoder_hidden(const lv_encoder *enc);

// Embed the token rows of node ids d_ids[0..count) of a token store
// (u16/u32 [n][seq_len]) into out[count][hidden] fp32 (unit norm).
int encode_node_rows(lv_encoder *enc, const void *tokens, int token_bytes, int seq_len,
                     const int32_t *d_ids, int64_t count, float *out, cudaStream_t s);

// Fold the GEMM events recorded in profile mode into the encoder's counters
// (call after the launching stream has been synchronised).
void encoder_collect_profile(lv_encoder *enc);

}  // namespace lv
