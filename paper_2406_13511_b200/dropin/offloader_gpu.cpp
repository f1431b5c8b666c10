// offloader_gpu.cpp — drop-in replacement of the reference's
// core/src/offloader.cpp: offload (offloader.h:39-40) on the B200 via
// scls_offload; complete_batch (offloader.h:44) is the scalar load update.
#include <utility>
#include <vector>

#include "dropin.h"
#include "slicesim/offloader.h"

namespace slicesim {

std::vector<std::pair<BatchId, WorkerId>> offload(const std::vector<Batch>& batches,
                                                  std::vector<WorkerLoad>& workers) {
  if (batches.empty()) return {};  // offloader.cpp:26: nothing to place, no worker check
  const int64_t nb = static_cast<int64_t>(batches.size());
  const int32_t nw = static_cast<int32_t>(workers.size());
  std::vector<int64_t> bid(nb), ob(nb);
  std::vector<double> est(nb), load(nw);
  std::vector<int32_t> wid(nw), ow(nb);
  for (int64_t b = 0; b < nb; ++b) {
    bid[b] = batches[b].id;
    est[b] = batches[b].est_serve_time;
  }
  for (int32_t w = 0; w < nw; ++w) {
    wid[w] = workers[w].worker_id;
    load[w] = workers[w].load_estimate;
  }
  scls_ctx* ctx = b200::context();
  b200::check(ctx, scls_offload(ctx, nb, bid.data(), est.data(), nw, wid.data(), load.data(), ob.data(),
                                ow.data(), SCLS_MEM_HOST));
  for (int32_t w = 0; w < nw; ++w) workers[w].load_estimate = load[w];
  std::vector<std::pair<BatchId, WorkerId>> out(static_cast<size_t>(nb));
  for (int64_t k = 0; k < nb; ++k) out[k] = {ob[k], ow[k]};
  return out;
}

void complete_batch(WorkerLoad& worker, double batch_est_s) {
  worker.load_estimate -= batch_est_s;
  if (worker.load_estimate < 0.0) worker.load_estimate = 0.0;
}

}  // namespace slicesim
