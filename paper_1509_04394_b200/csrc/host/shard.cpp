// Single-process multi-GPU execution of a plan over a T-sharded video: the
// C / C++ caller's entry point (fp_shard_exec_*, include/fuseplan.h).  The
// Python ranks of paper_1509_04394_b200/sharding.py run the same protocol one
// process per GPU over torch.distributed / NCCL; here one host thread drives
// every device and the carry plane moves device to device with
// cudaMemcpyPeerAsync (NVLink peer copies inside the node; a plain device copy
// when two "ranks" share a GPU, which is how it is tested on one B200).
//
// Protocol, exact for any warm-up length W:
//   rank g owns frames [lo_g, hi_g); it restarts the IIR W frames before lo_g
//   (the reference restarts at frame 0, simulator.cpp:136-147), keeps that
//   warm state, runs its shard and keeps the end state;
//   every carry s_end(g-1) is copied to rank g and checked against rank g's
//   warm state by fc_iir_converge, which returns k = the leading frames of
//   the shard whose IIR plane differs (the two trajectories coincide from
//   then on); if every k is 0 the output is exact (induction over the ranks);
//   else from the first such rank on, the carry walks the ranks in order and
//   each re-runs only frames [lo, lo + k) from the true state -- its end state
//   changes only when k reaches the shard's end, and only then does the walk
//   continue.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <functional>
#include <memory>
#include <sstream>
#include <vector>

#include "exec.hpp"

namespace fuseplan {

namespace {
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(ErrorKind::Internal, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

class ShardedExecutor {
 public:
  ShardedExecutor(const Pipeline& p, const FusionPlan& plan, std::vector<int> devices,
                  const ExecOptions& opt, int warmup)
      : dims_(p.video), devices_(std::move(devices)), warmup_(warmup) {
    require(!devices_.empty(), ErrorKind::Input, "sharded executor: no devices");
    require(warmup_ >= 0, ErrorKind::Input, "sharded executor: warmup_frames < 0");
    int n_dev = 0;
    ck(cudaGetDeviceCount(&n_dev), "cudaGetDeviceCount");
    for (int d : devices_)
      require(d >= 0 && d < n_dev, ErrorKind::Input, "device ordinal out of range");
    const int N = int(devices_.size());
    require(dims_.frames >= N, ErrorKind::Input, "fewer frames than shards");
    for (int g = 0; g < N; ++g) {
      Rank r;
      r.dev = devices_[g];
      r.lo = int((long long)g * dims_.frames / N);
      r.hi = int((long long)(g + 1) * dims_.frames / N);
      r.warm = std::min(warmup_, r.lo);
      r.ex = std::make_unique<Executor>(p, plan, r.dev, opt);
      ranks_.push_back(std::move(r));
    }
    require(ranks_[0].ex->iir_count() <= 1, ErrorKind::Input,
            "sharded executor: at most one IIR stage");
    // peer access between distinct devices (NVLink); same-device ranks copy locally
    for (int a : devices_)
      for (int b : devices_) {
        if (a == b) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, a, b);
        if (can) {
          cudaSetDevice(a);
          cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            ck(e, "cudaDeviceEnablePeerAccess");
          cudaGetLastError();
        }
      }
  }

  ~ShardedExecutor() {
    for (auto& r : ranks_) {
      cudaSetDevice(r.dev);
      for (void* p : {r.video, r.out, static_cast<void*>(r.s_warm), static_cast<void*>(r.s_end),
                      static_cast<void*>(r.s_true)})
        if (p) cudaFree(p);
      if (r.st) cudaStreamDestroy(r.st);
      if (r.done) cudaEventDestroy(r.done);
    }
  }

  // Host buffers in and out (planar [t][c][y][x] video, [t][y][x] output);
  // synchronous.
  void run(const void* video, int in_type, void* out) {
    const long long hw = (long long)dims_.width * dims_.height;
    const int C = dims_.channels;
    const size_t esz = in_type == FC_U8 ? 1 : 4;
    const int out_type = ranks_[0].ex->output_type();
    const size_t osz = out_type == FC_U8 ? 1 : 4;
    const bool has_iir = ranks_[0].ex->iir_count() == 1;
    stats_ = {};
    // 1. every rank: stage its frames (warm-up included), warm-up launch,
    //    shard launch -- all asynchronous, the devices run concurrently
    for (auto& r : ranks_) {
      ck(cudaSetDevice(r.dev), "cudaSetDevice");
      if (!r.st) {
        ck(cudaStreamCreateWithFlags(&r.st, cudaStreamNonBlocking), "stream");
        ck(cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming), "event");
      }
      const int n_in = r.hi - r.lo + r.warm;
      const size_t vbytes = size_t(n_in) * C * hw * esz, obytes = size_t(r.hi - r.lo) * hw * osz;
      if (vbytes > r.video_cap) {
        if (r.video) cudaFree(r.video);
        ck(cudaMalloc(&r.video, vbytes), "cudaMalloc(shard video)");
        r.video_cap = vbytes;
      }
      if (obytes > r.out_cap) {
        if (r.out) cudaFree(r.out);
        ck(cudaMalloc(&r.out, obytes), "cudaMalloc(shard out)");
        r.out_cap = obytes;
      }
      if (!r.s_end) {
        ck(cudaMalloc(&r.s_warm, hw * 4), "cudaMalloc(state)");
        ck(cudaMalloc(&r.s_end, hw * 4), "cudaMalloc(state)");
        ck(cudaMalloc(&r.s_true, hw * 4), "cudaMalloc(state)");
      }
      const char* src = static_cast<const char*>(video) + size_t(r.lo - r.warm) * C * hw * esz;
      ck(cudaMemcpyAsync(r.video, src, vbytes, cudaMemcpyHostToDevice, r.st), "H2D shard");
      if (r.warm)  // the IIR restarted W frames early: state only
        r.ex->run_device(r.video, in_type, nullptr, r.warm, r.warm, nullptr, r.s_warm, r.st);
      r.ex->run_device(static_cast<char*>(r.video) + size_t(r.warm) * C * hw * esz, in_type,
                       r.out, r.hi - r.lo, 0, r.warm ? r.s_warm : nullptr,
                       has_iir ? r.s_end : nullptr, r.st);
      ck(cudaEventRecord(r.done, r.st), "event");
    }
    // 2. carries: s_end(g-1) -> rank g (peer copy), then the convergence check
    if (has_iir) {
      for (size_t g = 1; g < ranks_.size(); ++g) {
        Rank &a = ranks_[g - 1], &b = ranks_[g];
        ck(cudaSetDevice(b.dev), "cudaSetDevice");
        ck(cudaStreamWaitEvent(b.st, a.done, 0), "wait carry");
        ck(cudaMemcpyPeerAsync(b.s_true, b.dev, a.s_end, a.dev, hw * 4, b.st), "carry copy");
      }
      std::vector<int> k(ranks_.size(), 0);
      for (size_t g = 1; g < ranks_.size(); ++g) k[g] = check(ranks_[g], in_type);
      // 3. fix-up walk in rank order: rank g's carry is final once every
      //    rank before it is; a fix-up that reaches the shard's end changes
      //    the end state, so the next rank's carry is re-sent and re-checked
      for (size_t g = 1; g < ranks_.size(); ++g) {
        Rank& r = ranks_[g];
        if (k[g] == 0) continue;  // this rank's warm state was the carry
        const int n_local = r.hi - r.lo;
        const bool whole = k[g] >= n_local;
        ck(cudaSetDevice(r.dev), "cudaSetDevice");
        r.ex->run_device(static_cast<char*>(r.video) + size_t(r.warm) * C * hw * esz, in_type,
                         r.out, std::min(k[g], n_local), 0, r.s_true,
                         whole ? r.s_end : nullptr, r.st);
        ++stats_.fixups;
        stats_.fixed_frames += std::min(k[g], n_local);
        if (!whole || g + 1 == ranks_.size()) continue;  // end state unchanged
        Rank& nx = ranks_[g + 1];
        ck(cudaEventRecord(r.done, r.st), "event");
        ck(cudaSetDevice(nx.dev), "cudaSetDevice");
        ck(cudaStreamWaitEvent(nx.st, r.done, 0), "wait carry");
        ck(cudaMemcpyPeerAsync(nx.s_true, nx.dev, r.s_end, r.dev, hw * 4, nx.st), "carry copy");
        k[g + 1] = check(nx, in_type);
      }
    }
    // 4. outputs back to the host
    for (auto& r : ranks_) {
      ck(cudaSetDevice(r.dev), "cudaSetDevice");
      ck(cudaMemcpyAsync(static_cast<char*>(out) + size_t(r.lo) * hw * osz, r.out,
                         size_t(r.hi - r.lo) * hw * osz, cudaMemcpyDeviceToHost, r.st),
         "D2H shard");
    }
    for (auto& r : ranks_) {
      ck(cudaSetDevice(r.dev), "cudaSetDevice");
      ck(cudaStreamSynchronize(r.st), "shard sync");
    }
    ++stats_.runs;
  }

  std::string stats() const {
    std::ostringstream ss;
    ss << "{\"shards\": " << ranks_.size() << ", \"warmup_frames\": " << warmup_
       << ", \"fixups\": " << stats_.fixups << ", \"fixed_frames\": " << stats_.fixed_frames
       << ", \"devices\": [";
    for (size_t i = 0; i < ranks_.size(); ++i)
      ss << (i ? ", " : "") << "{\"device\": " << ranks_[i].dev << ", \"frames\": ["
         << ranks_[i].lo << ", " << ranks_[i].hi << "], \"warm\": " << ranks_[i].warm << "}";
    ss << "]}";
    return ss.str();
  }

 private:
  struct Rank {
    int dev = 0, lo = 0, hi = 0, warm = 0;
    std::unique_ptr<Executor> ex;
    void* video = nullptr;
    size_t video_cap = 0;
    void* out = nullptr;
    size_t out_cap = 0;
    float* s_warm = nullptr;
    float* s_end = nullptr;
    float* s_true = nullptr;
    cudaStream_t st = nullptr;
    cudaEvent_t done = nullptr;
  };

  // leading frames of rank r's shard that its warm start got wrong
  int check(Rank& r, int in_type) {
    const long long hw = (long long)dims_.width * dims_.height;
    const size_t esz = in_type == FC_U8 ? 1 : 4;
    ck(cudaSetDevice(r.dev), "cudaSetDevice");
    if (r.warm == 0) {  // no warm-up: the shard started from a fresh recurrence
      // (only rank 0 starts fresh legitimately; any other rank is fully wrong)
      return r.hi - r.lo;
    }
    return r.ex->converge(static_cast<char*>(r.video) + size_t(r.warm) * dims_.channels * hw * esz,
                          in_type, r.hi - r.lo, r.s_true, r.s_warm, r.st);
  }

  VideoDims dims_;
  std::vector<int> devices_;
  int warmup_ = 48;
  std::vector<Rank> ranks_;
  struct {
    int runs = 0, fixups = 0;
    long long fixed_frames = 0;
  } stats_;
};

}  // namespace fuseplan

// ------------------------------------------------------------------ C ABI glue
// (declared in include/fuseplan.h; status / error conventions of capi.cpp)

#include "../../../include/fuseplan.h"

struct fp_shard_exec {
  std::unique_ptr<fuseplan::ShardedExecutor> ex;
};

namespace fuseplan {
// capi.cpp helpers
fp_status capi_guarded(const std::function<void()>& fn);
const Pipeline& capi_pipeline(const fp_pipeline* p);
const FusionPlan& capi_plan(const fp_plan* p);
ExecOptions capi_exec_options(const char* options_json, int* warmup_frames);
char* capi_dup(const std::string& s);
}  // namespace fuseplan

extern "C" {

fp_status fp_shard_exec_create(const fp_pipeline* p, const fp_plan* plan, const int* devices,
                               int n_devices, const char* options_json, fp_shard_exec** out) {
  using namespace fuseplan;
  return capi_guarded([&] {
    require(p && plan && devices && out && n_devices > 0, ErrorKind::Input, "null argument");
    int warm = 48;
    ExecOptions o = capi_exec_options(options_json, &warm);
    auto h = std::make_unique<fp_shard_exec>();
    h->ex = std::make_unique<ShardedExecutor>(capi_pipeline(p), capi_plan(plan),
                                              std::vector<int>(devices, devices + n_devices), o,
                                              warm);
    *out = h.release();
  });
}

void fp_shard_exec_free(fp_shard_exec* e) { delete e; }

fp_status fp_shard_exec_run(fp_shard_exec* e, const void* video, int in_type, void* out) {
  using namespace fuseplan;
  return capi_guarded([&] {
    require(e && video && out, ErrorKind::Input, "null argument");
    require(in_type == FP_ELEM_U8 || in_type == FP_ELEM_F32, ErrorKind::Input,
            "in_type must be FP_ELEM_U8 or FP_ELEM_F32");
    e->ex->run(video, in_type, out);
  });
}

fp_status fp_shard_exec_stats(const fp_shard_exec* e, char** out_json) {
  using namespace fuseplan;
  return capi_guarded([&] {
    require(e && out_json, ErrorKind::Input, "null argument");
    *out_json = capi_dup(e->ex->stats());
  });
}

}  // extern "C"
