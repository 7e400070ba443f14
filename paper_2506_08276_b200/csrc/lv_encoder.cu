// lv_encoder.cu — placeholder until the encoder lands.
#include "lv_encoder.cuh"

struct lv_encoder {
  int hidden = 0;
};

namespace lv {
int encoder_hidden(const lv_encoder *enc) { return enc ? enc->hidden : 0; }
int encode_node_rows(lv_encoder *, const void *, int, int, const int32_t *, int64_t, float *,
                     cudaStream_t) {
  set_error("encoder not available");
  return LV_ERR_INTERNAL;
}
}  // namespace lv

extern "C" {
int lv_encoder_create(const lv_encoder_config *, const float *const *, int32_t, int, lv_encoder **) {
  lv::set_error("encoder not available");
  return LV_ERR_INTERNAL;
}
void lv_encoder_destroy(lv_encoder *enc) { delete enc; }
int lv_encode(lv_encoder *, const void *, int32_t, int64_t, int32_t, float *, int, void *) {
  lv::set_error("encoder not available");
  return LV_ERR_INTERNAL;
}
}
