// batcher_gpu.cpp — drop-in replacement of the reference's core/src/batcher.cpp:
// batch_requests (batcher.h:40-43) on the B200 via scls_batch_requests.
// Same signature, same batches (ids, members in sorted order, l_in,
// planned_l_out, est_serve_time bit for bit), same InfeasibleRequestError.
#include <vector>

#include "dropin.h"
#include "slicesim/batcher.h"

namespace slicesim {

std::vector<Batch> batch_requests(const std::vector<Request>& requests, int slice_len,
                                  const LatencyModel& latency, const MemoryModel& memory,
                                  BatchId first_batch_id) {
  if (requests.empty()) return {};
  const int64_t n = static_cast<int64_t>(requests.size());
  std::vector<int32_t> eff(n);
  std::vector<double> arrival(n);
  std::vector<int64_t> id(n);
  for (int64_t i = 0; i < n; ++i) {
    eff[i] = requests[i].effective_input_len();
    arrival[i] = requests[i].arrival_time;
    id[i] = requests[i].id;
  }
  std::vector<int32_t> seg(n + 1), l_in(n);
  std::vector<double> est(n);
  std::vector<int64_t> member(n);
  scls_batches out{0, nullptr, seg.data(), l_in.data(), est.data(), member.data()};
  const scls_latency lat = b200::to_c(latency);
  const scls_memory mem = b200::to_c(memory);
  scls_ctx* ctx = b200::context();
  b200::check(ctx, scls_batch_requests(ctx, n, eff.data(), arrival.data(), id.data(), slice_len, &lat, &mem,
                                       first_batch_id, &out, SCLS_MEM_HOST));
  std::vector<Batch> batches(static_cast<size_t>(out.n_batches));
  for (int64_t b = 0; b < out.n_batches; ++b) {
    Batch& bt = batches[b];
    bt.id = first_batch_id + b;
    bt.l_in = l_in[b];
    bt.planned_l_out = slice_len;
    bt.est_serve_time = est[b];
    bt.requests.assign(member.begin() + seg[b], member.begin() + seg[b + 1]);
  }
  return batches;
}

}  // namespace slicesim
