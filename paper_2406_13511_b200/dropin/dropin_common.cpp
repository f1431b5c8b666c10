// dropin_common.cpp — context, error mapping and struct conversion for the
// B200 drop-in (see dropin.h).
#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "dropin.h"

namespace slicesim {
namespace b200 {

namespace {
struct CtxHolder {
  scls_ctx* ctx = nullptr;
  ~CtxHolder() {
    if (ctx) scls_ctx_destroy(ctx);
  }
};
thread_local CtxHolder g_ctx;

std::string last_error(scls_ctx* ctx) {
  char buf[1024];
  scls_last_error(ctx, buf, sizeof buf);
  return buf;
}
}  // namespace

scls_ctx* context() {
  if (!g_ctx.ctx) {
    const char* env = std::getenv("SCLS_DEVICE");
    const int dev = env ? std::atoi(env) : 0;
    scls_ctx* c = nullptr;
    const scls_status st = scls_ctx_create(dev, nullptr, &c);
    if (st != SCLS_OK) throw Error("B200 scheduling core unavailable: " + last_error(nullptr));
    g_ctx.ctx = c;
  }
  return g_ctx.ctx;
}

namespace {
struct MultiHolder {
  scls_multi* m = nullptr;
  bool tried = false;
  ~MultiHolder() {
    if (m) scls_multi_destroy(m);
  }
};
thread_local MultiHolder g_multi;
}  // namespace

// Every visible GPU (SCLS_DEVICES=k limits it to devices 0..k-1); null when
// there is only one, so single-GPU callers keep the plain context.
scls_multi* multi() {
  if (!g_multi.tried) {
    g_multi.tried = true;
    const int count = scls_device_count();
    std::vector<int32_t> devs;
    const char* env = std::getenv("SCLS_DEVICES");
    if (env && std::string(env).find(',') != std::string::npos) {  // an explicit list, e.g. "0,1" or "0,0"
      std::string s(env);
      for (size_t p = 0; p <= s.size();) {
        const size_t q = std::min(s.find(',', p), s.size());
        devs.push_back(std::atoi(s.substr(p, q - p).c_str()));
        p = q + 1;
      }
    } else {
      const int n = env ? std::min(count, std::atoi(env)) : count;
      for (int i = 0; i < n; ++i) devs.push_back(i);
    }
    if (devs.size() > 1) {
      scls_multi* m = nullptr;
      if (scls_multi_create((int32_t)devs.size(), devs.data(), &m) != SCLS_OK)
        throw Error("B200 multi-GPU sweep unavailable: " + last_error(nullptr));
      scls_multi_set_option(m, SCLS_OPT_SIM_DIGESTS, 0);  // sweeps report metrics only
      g_multi.m = m;
    }
  }
  return g_multi.m;
}

void raise(scls_ctx* ctx, scls_status st) {
  const std::string msg = last_error(ctx);
  switch (st) {
    case SCLS_ERR_INFEASIBLE_REQUEST: throw InfeasibleRequestError(scls_last_request_id(ctx), msg);
    case SCLS_ERR_NO_WORKERS: throw NoWorkersError(msg);
    case SCLS_ERR_NON_TERMINATION: throw NonTerminationError(msg);
    case SCLS_ERR_DEGENERATE_MODEL: throw DegenerateModelError(msg);
    case SCLS_ERR_WRONG_KIND: throw WrongKindError(msg);
    case SCLS_ERR_INSUFFICIENT_SAMPLES: throw InsufficientSamplesError(msg);
    case SCLS_ERR_EMPTY_LOG: throw EmptyLogError(msg);
    case SCLS_ERR_PARSE: throw ParseError(1, msg);
    case SCLS_ERR_LIMIT_VIOLATION: throw LimitViolationError(1, msg);
    default: throw Error(msg.empty() ? "B200 scheduling core error " + std::to_string(st) : msg);
  }
}

scls_latency to_c(const LatencyModel& m) {
  return scls_latency{m.p1, m.p2, m.p3, m.p4, m.d1, m.d2, m.d3, m.d4,
                      m.rmse_prefill, m.rmse_decode, m.n_cap, m.l_cap};
}

scls_memory to_c(const MemoryModel& m) {
  scls_memory c{};
  if (m.kind == MemoryModel::Kind::kAnalytic) {
    c.kind = SCLS_MEM_ANALYTIC;
    c.m_cap = m.m_cap;
    c.m_model = m.m_model;
    c.m_engine = m.m_engine;
    c.delta = m.delta;
    c.zeta = m.zeta;
  } else {
    if (m.rules.size() > SCLS_MAX_RULES)
      throw Error("B200 drop-in supports at most " + std::to_string(SCLS_MAX_RULES) + " rule-table rows");
    c.kind = SCLS_MEM_RULE_TABLE;
    c.n_rules = static_cast<int32_t>(m.rules.size());
    for (size_t i = 0; i < m.rules.size(); ++i) {
      c.rule_threshold[i] = m.rules[i].total_len_threshold;
      c.rule_max_n[i] = m.rules[i].max_batch_size;
    }
  }
  return c;
}

scls_sched_cfg to_c(const SchedulerConfig& c, double horizon_s) {
  scls_sched_cfg r{};
  r.policy = c.policy == PolicyKind::kScls ? SCLS_POLICY_SCLS
             : c.policy == PolicyKind::kSls ? SCLS_POLICY_SLS
                                            : SCLS_POLICY_ILS;
  r.slice_len = c.slice_len;
  r.max_gen_limit = c.max_gen_limit;
  r.fixed_batch_size = c.fixed_batch_size;
  r.max_concurrent = c.max_concurrent;
  r.worker_count = c.worker_count;
  r.lambda = c.lambda;
  r.gamma = c.gamma;
  r.horizon_s = horizon_s;
  return r;
}

}  // namespace b200
}  // namespace slicesim
