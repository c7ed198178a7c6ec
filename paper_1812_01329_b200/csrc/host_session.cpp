// host_session.cpp — graph cache + relaxation driver (janus.h "Graph
// cache + relaxation driver").
//
// Figure 2 of the paper as a host state machine around janus_graph_build / janus_run /
// janus_run_imperative: graphs are cached with the assumptions they were generated under
// (P:154), looked up by their DISPATCH assumptions (a mismatch is a cache miss served
// imperatively), an AssertOp failure falls back to the imperative executor, and an
// assumption that "repeatedly breaks" is relaxed one level of the Figure 4 hierarchy
// and the graph regenerated. Threshold 2 and the per-key dispatch polymorphism follow
// SPEC's orchestrator. Host code only; the device work is whatever the dispatched
// graph or the imperative executor launches.
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "host.h"

using namespace jk;

namespace {

struct Entry {
  int id = 0;
  std::vector<janus_assumption> asms;
  janus_graph *g = nullptr;
  bool device = false;  // janus_graph_build returned OK (else: imperative-only entry)
  bool active = true;
  uint64_t hits = 0, last_use = 0;
  std::map<uint32_t, int> fails;  // committed-fallback failures per assumption id
  std::string origin;             // "initial" | "relax:<id>" | "miss:<key>"
};

std::string key_of(const janus_failure &f, const janus_tensor &t) {
  char b[160];
  snprintf(b, sizeof b, "%u:dt%d:nd%d:%lld,%lld,%lld,%lld", f.assumption_id, t.dtype, t.ndim,
           (long long)t.shape[0], (long long)t.shape[1], (long long)t.shape[2],
           (long long)t.shape[3]);
  return b;
}

const char *kind_name(int k) {
  static const char *n[] = {"DTYPE_EQ", "SHAPE_MATCH", "TRIP_COUNT", "TYPE_TAG",
                            "RANGE",    "TREE_BINARY", "VALUE_EQ",   "BRANCH_ARM"};
  return k >= 0 && k <= 7 ? n[k] : "?";
}

std::string asm_text(const janus_assumption &a) {
  char b[200];
  switch (a.kind) {
    case JA_DTYPE_EQ: snprintf(b, sizeof b, "%u:%s(arg%d,dt%d)", a.id, kind_name(a.kind), a.target, a.dtype); break;
    case JA_SHAPE_MATCH: {
      std::string d;
      for (int k = 0; k < a.ndim && k < 4; ++k) {
        if (k) d += ",";
        d += a.dims[k] < 0 ? std::string("?") : std::to_string(a.dims[k]);
      }
      snprintf(b, sizeof b, "%u:%s(arg%d,(%s))", a.id, kind_name(a.kind), a.target, d.c_str());
      break;
    }
    case JA_RANGE:
      snprintf(b, sizeof b, "%u:%s(arg%d,[%lld,%lld])", a.id, kind_name(a.kind), a.target,
               (long long)a.lo, (long long)a.hi);
      break;
    default:
      snprintf(b, sizeof b, "%u:%s(%d,%lld)", a.id, kind_name(a.kind), a.target, (long long)a.value);
  }
  return b;
}

// DISPATCH check of an assumption vector without a graph (same rule as check_dispatch).
bool dispatch_ok(const std::vector<janus_assumption> &asms, const janus_tensor *args, int n_args,
                 janus_failure *fail) {
  Graph tmp;
  tmp.asms = asms;
  tmp.opts.fail_assert_id = -1;
  return check_dispatch(tmp, args, n_args, fail);
}

}  // namespace

struct janus_session {
  std::vector<janus_op> ops;
  janus_build_opts bopts{};
  int threshold = 2, cache_max = 0;
  std::vector<Entry> entries;  // creation order; retired entries keep their record (graph freed)
  janus_graph *generic = nullptr;
  std::map<std::string, int> miss_count;
  uint64_t calls = 0, graph_calls = 0, imp_calls = 0, misses = 0, generated = 0, clock = 0;
  std::map<uint32_t, uint64_t> aborts;
  const void *ws_last_graph = nullptr;  // graph that last ran on the workspace

  int build(std::vector<janus_assumption> asms, const std::string &origin) {
    Entry e;
    e.id = (int)entries.size();
    e.asms = std::move(asms);
    e.origin = origin;
    janus_graph *g = nullptr;
    janus_status r = janus_graph_build(ops.data(), (int32_t)ops.size(), e.asms.data(),
                                       (int32_t)e.asms.size(), &bopts, &g, nullptr, 0);
    if (r != JANUS_OK && r != JANUS_ERR_UNSUPPORTED) {
      janus_graph_destroy(g);
      return -1;
    }
    e.g = g;
    e.device = r == JANUS_OK;
    e.last_use = clock;
    entries.push_back(std::move(e));
    generated++;
    evict();
    return (int)entries.size() - 1;
  }
  void retire(Entry &e) {
    if (!e.active) return;
    e.active = false;
    if (ws_last_graph == e.g) ws_last_graph = nullptr;
    janus_graph_destroy(e.g);
    e.g = nullptr;
  }
  void evict() {
    if (cache_max <= 0) return;
    for (;;) {
      int n = 0, lru = -1;
      for (int i = 0; i < (int)entries.size(); ++i)
        if (entries[i].active) {
          ++n;
          if (i + 1 < (int)entries.size() && (lru < 0 || entries[i].last_use < entries[lru].last_use)) lru = i;
        }
      if (n <= cache_max || lru < 0) return;
      retire(entries[lru]);
    }
  }
  // the step's workspace is shared by every entry: a graph must not trust a workspace another
  // graph (or the imperative executor) wrote since its last run
  void bind_workspace(janus_graph *g) {
    if (ws_last_graph != g) g->ws_ready = nullptr;  // janus_run re-initialises it
    ws_last_graph = g;
  }
};

namespace {

// Specialise `base` to the arguments it missed on: every failing DISPATCH assumption is replaced
// by janus_relax (join == true: per-dim join for shapes) or by the exact observed key.
std::vector<janus_assumption> specialise(const std::vector<janus_assumption> &base,
                                         const janus_tensor *args, int n_args, bool join,
                                         bool *dtype_changed) {
  std::vector<janus_assumption> v = base;
  *dtype_changed = false;
  for (size_t it = 0; it <= v.size(); ++it) {
    janus_failure f{};
    if (dispatch_ok(v, args, n_args, &f)) break;
    auto p = std::find_if(v.begin(), v.end(), [&](const janus_assumption &a) { return a.id == f.assumption_id; });
    if (p == v.end()) break;
    if (p->target < 0 || p->target >= n_args) { v.erase(p); continue; }
    const janus_tensor &t = args[p->target];
    if (p->kind == JA_DTYPE_EQ) {
      p->dtype = t.dtype;
      *dtype_changed = true;
    } else if (p->kind == JA_SHAPE_MATCH) {
      if (join) {
        janus_assumption o{};
        int32_t dropped = 0;
        janus_relax(&*p, &t, &o, &dropped);
        if (dropped) v.erase(p);
        else *p = o;
      } else {
        p->ndim = std::min(t.ndim, 4);
        for (int k = 0; k < 4; ++k) p->dims[k] = k < t.ndim ? t.shape[k] : 0;
      }
    } else {
      v.erase(p);
    }
  }
  // A dim joined to '?' makes the batch width vary, so an exact trip count cannot hold for every
  // key the joined graph serves: the loop is relaxed with it (TRIP_COUNT -> RANGE [1, n], a
  // bounded device While, Figure 4 one level up) instead of staying unrolled to the old width.
  bool widened = false;
  for (const auto &a : v)
    if (a.kind == JA_SHAPE_MATCH)
      for (const auto &b0 : base)
        if (b0.id == a.id)
          for (int k = 0; k < a.ndim && k < 4; ++k) widened |= a.dims[k] < 0 && b0.dims[k] >= 0;
  if (join && widened)
    for (auto &a : v)
      if (a.kind == JA_TRIP_COUNT) {
        janus_assumption o{};
        int32_t dropped = 0;
        if (janus_relax(&a, nullptr, &o, &dropped) == JANUS_OK && !dropped) a = o;
      }
  return v;
}

}  // namespace

extern "C" {

janus_status janus_relax(const janus_assumption *a, const janus_tensor *observed,
                         janus_assumption *out, int32_t *dropped) {
  if (!a || !out || !dropped) return JANUS_ERR_INVALID;
  *dropped = 0;
  switch (a->kind) {
    case JA_DTYPE_EQ:
      if (!observed) return JANUS_ERR_INVALID;
      *out = *a;
      out->dtype = observed->dtype;
      return JANUS_OK;
    case JA_SHAPE_MATCH:
      if (!observed) return JANUS_ERR_INVALID;
      if (observed->ndim != a->ndim) { *dropped = 1; return JANUS_OK; }
      *out = *a;
      for (int k = 0; k < a->ndim && k < 4; ++k)
        if (a->dims[k] != observed->shape[k]) out->dims[k] = -1;
      return JANUS_OK;
    case JA_TRIP_COUNT:
      *out = *a;
      out->kind = JA_RANGE;
      out->lo = 1;
      out->hi = a->value;
      out->value = 0;
      out->ref_arg = -1;
      out->ref_dim = -1;
      return JANUS_OK;
    case JA_TYPE_TAG: case JA_VALUE_EQ: case JA_BRANCH_ARM: case JA_RANGE: case JA_TREE_BINARY:
      *dropped = 1;
      return JANUS_OK;
  }
  return JANUS_ERR_INVALID;
}

janus_status janus_session_create(const janus_op *ops, int32_t n_ops, const janus_assumption *asms,
                                  int32_t n_asms, const janus_build_opts *bopts,
                                  const janus_session_opts *opts, janus_session **out, char *err,
                                  size_t err_len) {
  if (!out) return JANUS_ERR_INVALID;
  *out = nullptr;
  if (bopts && bopts->world_size > 1) {
    if (err && err_len) snprintf(err, err_len, "sessions are single-GPU (world_size 1)");
    return JANUS_ERR_UNSUPPORTED;
  }
  janus_session *s = new janus_session();
  if (bopts) s->bopts = *bopts;
  else {
    s->bopts.world_size = 1;
    s->bopts.gemm_dtype = JANUS_BF16;
    s->bopts.fail_assert_id = -1;
  }
  if (opts && opts->fail_threshold > 0) s->threshold = opts->fail_threshold;
  if (opts && opts->cache_max > 0) s->cache_max = opts->cache_max;
  // the initial entry: the caller's assumptions (validation errors are reported here)
  janus_graph *g0 = nullptr;
  janus_status r = janus_graph_build(ops, n_ops, asms, n_asms, &s->bopts, &g0, err, err_len);
  if (r != JANUS_OK && r != JANUS_ERR_UNSUPPORTED) {
    delete s;
    return r;
  }
  s->ops.assign(ops, ops + n_ops);
  Entry e;
  e.id = 0;
  e.asms.assign(asms, asms + n_asms);
  e.g = g0;
  e.device = r == JANUS_OK;
  e.origin = "initial";
  s->entries.push_back(std::move(e));
  // the miss path: the generic program without assumptions (imperative executor only)
  if (janus_graph_build(ops, n_ops, nullptr, 0, &s->bopts, &s->generic, nullptr, 0) != JANUS_ERR_UNSUPPORTED &&
      !s->generic) {
    janus_session_destroy(s);
    return JANUS_ERR_INVALID;
  }
  *out = s;
  return r;
}

janus_status janus_session_workspace_bytes(const janus_session *s, size_t *bytes) {
  if (!s || !bytes) return JANUS_ERR_INVALID;
  size_t m = s->generic ? s->generic->ws_bytes : 0;
  for (const auto &e : s->entries)
    if (e.active && e.g) m = std::max(m, e.g->ws_bytes);
  *bytes = m;
  return JANUS_OK;
}

static size_t ws_size(const janus_tensor &ws) {
  return ws.data ? (size_t)ws.shape[0] * (ws.dtype == JANUS_U8 ? 1 : 4) : 0;
}

janus_status janus_session_step(janus_session *s, const janus_tensor *args, int32_t n_args,
                                const janus_tensor *state, int32_t n_state,
                                const janus_tensor *outs, int32_t n_outs, janus_tensor workspace,
                                void *cuda_stream, janus_step_info *info) {
  janus_step_info loc;
  if (!info) info = &loc;
  memset(info, 0, sizeof *info);
  info->entry = -1;
  info->generated = -1;
  if (!s || (!args && n_args) || (!state && n_state)) return JANUS_ERR_INVALID;
  // 1. dispatch: the first active entry whose DISPATCH assumptions hold
  int hit = -1;
  janus_failure miss{};
  bool have_miss = false;
  for (int i = 0; i < (int)s->entries.size(); ++i) {
    Entry &e = s->entries[i];
    if (!e.active) continue;
    janus_failure f{};
    if (check_dispatch(*e.g, args, n_args, &f)) { hit = i; break; }
    if (!have_miss) { miss = f; have_miss = true; }
  }
  janus_graph *run_g = hit >= 0 ? s->entries[hit].g : s->generic;
  info->workspace_bytes = run_g->ws_bytes;
  if (ws_size(workspace) < run_g->ws_bytes) return JANUS_ERR_WORKSPACE;
  s->calls++;
  s->clock++;
  auto imperative = [&](janus_graph *g) {
    s->imp_calls++;
    info->path = JANUS_PATH_IMPERATIVE;
    s->bind_workspace(g);
    return janus_run_imperative(g, args, n_args, state, n_state, outs, n_outs, workspace, cuda_stream);
  };
  if (hit < 0) {
    // 2a. cache miss: imperative; a key that keeps missing gets its own graph
    s->misses++;
    info->event = JANUS_EV_MISS;
    info->fail = miss;
    const janus_status r = imperative(s->generic);
    if (r == JANUS_OK && have_miss && miss.assumption_id != 0xffffffffu) {
      const janus_assumption *a = nullptr;
      int base = -1;
      for (int i = 0; i < (int)s->entries.size() && base < 0; ++i)
        if (s->entries[i].active) base = i;
      // every entry may have been evicted (cache_max): specialise the initial assumptions, whose
      // record is kept after retirement
      const std::vector<janus_assumption> base_asms = s->entries[base >= 0 ? base : 0].asms;
      for (const auto &x : base_asms)
        if (x.id == miss.assumption_id) a = &x;
      if (a && a->target >= 0 && a->target < n_args &&
          ++s->miss_count[key_of(miss, args[a->target])] >= s->threshold) {
        bool dt = false;
        std::vector<janus_assumption> joined = specialise(base_asms, args, n_args, true, &dt);
        int id = -1;
        if (!dt) {
          // shapes only: the Figure 4 join ("(4,8) and (3,8)" -> "(?,8)") generates
          // another graph that serves the new key; the older, more specialised entry stays in
          // front of it in dispatch order and keeps serving its own key (it is never retired on
          // the assumption that the joined plan can run it). A joined graph without a device
          // program is dropped in favour of an exact-key graph.
          id = s->build(joined, "miss-join");
          if (id >= 0 && !s->entries[id].device) { s->retire(s->entries[id]); id = -1; }
        }
        if (id < 0) id = s->build(specialise(base_asms, args, n_args, false, &dt), "miss-key");
        info->generated = id;
      }
    }
    return r;
  }
  // 2b. dispatched
  Entry &e = s->entries[hit];
  e.hits++;
  e.last_use = s->clock;
  info->entry = e.id;
  if (!e.device) {
    info->event = JANUS_EV_IMPERATIVE_ENTRY;
    return imperative(e.g);
  }
  s->bind_workspace(e.g);
  janus_failure f{};
  const janus_status r = janus_run(e.g, args, n_args, state, n_state, outs, n_outs, workspace,
                                   cuda_stream, &f);
  if (r == JANUS_OK) {
    s->graph_calls++;
    info->path = JANUS_PATH_GRAPH;
    info->event = JANUS_EV_HIT;
    return r;
  }
  if (r == JANUS_ERR_INVALID || r == JANUS_ERR_UNSUPPORTED) {
    // the device program cannot take THESE arguments (e.g. a joined '?' dim beyond the width it
    // was lowered for): nothing ran; this call is served imperatively, the entry keeps its
    // device program for the keys it can run
    info->event = JANUS_EV_IMPERATIVE_ENTRY;
    return imperative(e.g);
  }
  if (r != JANUS_ASSUMPTION_FAILED) return r;  // ERR_RUNTIME / ERR_CUDA: nothing committed
  // 3. AssertOp failure: the imperative result of the same step
  s->aborts[f.assumption_id]++;
  info->event = JANUS_EV_ABORT;
  info->fail = f;
  const janus_status ri = imperative(e.g);
  if (ri == JANUS_OK && ++e.fails[f.assumption_id] >= s->threshold) {
    std::vector<janus_assumption> v = e.asms;
    auto p = std::find_if(v.begin(), v.end(), [&](const janus_assumption &a) { return a.id == f.assumption_id; });
    if (p != v.end()) {
      janus_assumption o{};
      int32_t dropped = 0;
      const janus_tensor *obs = p->target >= 0 && p->target < n_args ? &args[p->target] : nullptr;
      if (janus_relax(&*p, obs, &o, &dropped) == JANUS_OK) {
        if (dropped) v.erase(p);
        else *p = o;
        const int id = s->build(v, "relax:" + std::to_string(f.assumption_id));
        if (id >= 0) {
          // the other assumptions keep their failure history (S:520 per-assumption counts)
          s->entries[id].fails = s->entries[hit].fails;
          s->entries[id].fails.erase(f.assumption_id);
          s->retire(s->entries[hit]);  // (entries may have reallocated: index again)
          info->generated = id;
        }
      }
    }
  }
  return ri;
}

janus_status janus_session_stats(const janus_session *s, char *buf, size_t buf_len) {
  if (!s || !buf || !buf_len) return JANUS_ERR_INVALID;
  std::string j = "{";
  char t[256];
  snprintf(t, sizeof t,
           "\"calls\": %llu, \"graph_calls\": %llu, \"imperative_calls\": %llu, \"misses\": %llu, "
           "\"generated\": %llu, \"fail_threshold\": %d, \"aborts\": {",
           (unsigned long long)s->calls, (unsigned long long)s->graph_calls,
           (unsigned long long)s->imp_calls, (unsigned long long)s->misses,
           (unsigned long long)s->generated, s->threshold);
  j += t;
  bool first = true;
  for (const auto &kv : s->aborts) {
    snprintf(t, sizeof t, "%s\"%u\": %llu", first ? "" : ", ", kv.first, (unsigned long long)kv.second);
    j += t;
    first = false;
  }
  j += "}, \"entries\": [";
  for (size_t i = 0; i < s->entries.size(); ++i) {
    const Entry &e = s->entries[i];
    snprintf(t, sizeof t, "%s{\"id\": %d, \"active\": %s, \"device\": %s, \"hits\": %llu, \"origin\": \"%s\", \"assumptions\": [",
             i ? ", " : "", e.id, e.active ? "true" : "false", e.device ? "true" : "false",
             (unsigned long long)e.hits, e.origin.c_str());
    j += t;
    for (size_t k = 0; k < e.asms.size(); ++k) j += (k ? ", \"" : "\"") + asm_text(e.asms[k]) + "\"";
    j += "]}";
  }
  j += "]}";
  if (j.size() + 1 > buf_len) return JANUS_ERR_INVALID;
  memcpy(buf, j.c_str(), j.size() + 1);
  return JANUS_OK;
}

void janus_session_destroy(janus_session *s) {
  if (!s) return;
  for (auto &e : s->entries) janus_graph_destroy(e.g);
  janus_graph_destroy(s->generic);
  delete s;
}

}  // extern "C"
