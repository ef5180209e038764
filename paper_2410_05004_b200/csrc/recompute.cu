// recompute.cu -- K6: the RECOMPUTE complement (prefill_layers).
#include "recompute.h"

namespace hc {

void prefill_layers_impl(const hc_weights* w, const int32_t* d_tokens, int64_t n, int lb, int le,
                         const hc_kv_pages* pages, const int32_t* d_page_table,
                         cudaStream_t stream, const std::function<void(int, bool)>& hook,
                         void* d_layer_inputs, int32_t* next_token) {
  (void)w; (void)d_tokens; (void)n; (void)lb; (void)le; (void)pages; (void)d_page_table;
  (void)stream; (void)hook; (void)d_layer_inputs; (void)next_token;
  fail(HC_ERUNTIME, "recompute path not built yet");
}

double recompute_layer_seconds(const hc_weights* w, int n) {
  (void)w;
  (void)n;
  return 0.0;
}

}  // namespace hc

using namespace hc;

extern "C" {

hc_status hc_prefill_layers(const hc_weights* w, const int32_t* d_tokens, int64_t n,
                            int32_t layer_begin, int32_t layer_end, const hc_kv_pages* pages,
                            const int32_t* d_page_table, void* stream) {
  return guard([&] {
    prefill_layers_impl(w, d_tokens, n, layer_begin, layer_end, pages, d_page_table,
                        as_stream(stream), [](int, bool) {});
  });
}

hc_status hc_prefill(const hc_weights* w, const int32_t* d_tokens, int64_t n,
                     const hc_kv_pages* pages, const int32_t* d_page_table, void* d_layer_inputs,
                     int32_t* next_token, void* stream) {
  return guard([&] {
    if (!w) fail(HC_EINVAL, "prefill: null weights");
    prefill_layers_impl(w, d_tokens, n, 0, w->cfg.n_layers, pages, d_page_table,
                        as_stream(stream), [](int, bool) {}, d_layer_inputs, next_token);
  });
}

}  // extern "C"
