// host_imperative.cpp — imperative per-op executor (placeholder).
#include "host.h"
namespace jk {
size_t imperative_ws_bytes(const Graph &) { return 0; }
janus_status run_imperative(Graph &, const janus_tensor *, int, const janus_tensor *, int,
                            const janus_tensor *, int, const janus_tensor &, cudaStream_t) {
  return JANUS_ERR_UNSUPPORTED;
}
}  // namespace jk
