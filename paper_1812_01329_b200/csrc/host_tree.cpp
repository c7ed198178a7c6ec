// host_tree.cpp — TreeLSTM lowering (placeholder until the level-batched program lands).
#include "host.h"
namespace jk {
bool lower_tree(Graph &g, std::string &why) { (void)g; why = "tree lowering not built yet"; return false; }
janus_status run_tree(Graph &, const janus_tensor *, int, const janus_tensor *, const janus_tensor *,
                      int, const janus_tensor &, cudaStream_t, janus_failure *) {
  return JANUS_ERR_UNSUPPORTED;
}
}  // namespace jk
