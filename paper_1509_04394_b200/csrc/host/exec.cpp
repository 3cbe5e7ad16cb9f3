// GPU executor (see exec.hpp).
#include "exec.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <cmath>
#include <cstring>
#include <sstream>

namespace fuseplan {

namespace {

void cuda_check(int rc, const char* what) {
  if (rc == 0) return;
  throw Error(ErrorKind::Internal, std::string(what) + ": " + fc_error_string(rc));
}

void cuda_check(cudaError_t rc, const char* what) { cuda_check(int(rc), what); }

double param(const KernelDesc& k, const char* key, double fallback) {
  auto it = k.params.find(key);
  return it == k.params.end() ? fallback : it->second;
}

int op_code(const std::string& op) {
  static const char* names[] = {"rgba2gray", "iir_temporal", "gaussian",
                                "gradient",  "threshold",    "identity",
                                "scale_offset", "box_mean"};
  for (int i = 0; i < 8; ++i)
    if (op == names[i]) return i;
  return -1;
}

bool is_byte_level(float v) {
  return v >= 0.0f && v <= 255.0f && v == std::floor(v);
}

struct Scratch {
  float* a;
  float* b;
};

// Value-range propagation for the certified F345 kernel (inputs must lie in
// [0, max]): nonnegative-weight averages keep the bound, everything else
// makes it unknown (-1).
double stage_range(const fc_stage& s, double in_max) {
  if (in_max < 0) return -1.0;
  switch (s.op) {
    case FC_RGBA2GRAY:
      if (s.wr < 0 || s.wg < 0 || s.wb < 0) return -1.0;
      return in_max * (double(s.wr) + double(s.wg) + double(s.wb));
    case FC_IIR_TEMPORAL:
      return (s.alpha >= 0.0f && s.alpha <= 1.0f) ? in_max : -1.0;
    case FC_IDENTITY:
    case FC_BOX_MEAN:
      return in_max;
    default:
      return -1.0;
  }
}

}  // namespace

std::vector<float> gaussian_taps(int radius, double sigma) {
  const int d = 2 * radius + 1;
  std::vector<double> raw(std::size_t(d) * d);
  double norm = 0.0;
  std::size_t i = 0;
  for (int dy = -radius; dy <= radius; ++dy)
    for (int dx = -radius; dx <= radius; ++dx, ++i) {
      raw[i] = std::exp(-(dx * dx + dy * dy) / (2.0 * sigma * sigma));
      norm += raw[i];
    }
  std::vector<float> taps(raw.size());
  for (std::size_t j = 0; j < raw.size(); ++j) taps[j] = float(raw[j] / norm);
  return taps;
}

fc_stage make_stage(const KernelDesc& k) {
  fc_stage s;
  std::memset(&s, 0, sizeof s);
  s.op = op_code(k.stencil_op);
  require(s.op >= 0, ErrorKind::Input,
          "stencil_op '" + k.stencil_op + "' has no device kernel");
  switch (s.op) {
    case FC_RGBA2GRAY:
      s.wr = float(param(k, "wr", 0.299));
      s.wg = float(param(k, "wg", 0.587));
      s.wb = float(param(k, "wb", 0.114));
      break;
    case FC_IIR_TEMPORAL:
      s.alpha = float(param(k, "alpha", 0.5));
      break;
    case FC_GAUSSIAN: {
      s.g_radius = int(param(k, "radius", 2));
      require(s.g_radius >= 0 && s.g_radius <= FC_MAX_GAUSS_RADIUS, ErrorKind::Input,
              "gaussian radius > " + std::to_string(FC_MAX_GAUSS_RADIUS) +
                  " has no device kernel");
      auto taps = gaussian_taps(s.g_radius, param(k, "sigma", 1.0));
      std::copy(taps.begin(), taps.end(), s.g_w);
      break;
    }
    case FC_THRESHOLD:
      s.th = float(param(k, "th", 128.0));
      s.white = float(param(k, "white", 255.0));
      s.black = float(param(k, "black", 0.0));
      break;
    case FC_SCALE_OFFSET:
      s.scale = float(param(k, "scale", 1.0));
      s.offset = float(param(k, "offset", 0.0));
      break;
    case FC_BOX_MEAN:
      s.rx = int(param(k, "radius_x", 1));
      s.ry = int(param(k, "radius_y", 1));
      s.rt = int(param(k, "radius_t", 0));
      break;
    default:
      break;
  }
  return s;
}

const char* LaunchGroup::kernel_name() const {
  switch (kind) {
    case GrayIir: return "F12 gray+iir (time scan)";
    case GaussGradThr: return "F345 gauss+grad+thr (certified frame pipeline / exact tiles)";
    case Chain: return "F12345 streaming chain (certified frame pipeline / exact)";
    default: return "unfused stages";
  }
}

Executor::Executor(const Pipeline& p, const FusionPlan& fp, int device,
                   const ExecOptions& opt)
    : device_(device), dims_(p.video), opt_(opt) {
  fc_knobs_from_env(&knobs_);
  int n_dev = 0;
  cudaError_t e = cudaGetDeviceCount(&n_dev);
  require(e == cudaSuccess && n_dev > 0, ErrorKind::Internal,
          std::string("no CUDA device available: ") + cudaGetErrorString(e));
  require(device >= 0 && device < n_dev, ErrorKind::Input,
          "device ordinal out of range");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cudaStream_t s;
  cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  own_stream_ = s;

  bool first = true;
  for (const PlanGroup& g : fp.groups) {
    if (g.global_aggregation) continue;  // tracking stage runs on the host
    LaunchGroup lg;
    lg.first = g.first;
    lg.last = g.last;
    std::vector<std::string> ops;
    for (int id = g.first; id <= g.last; ++id) {
      const KernelDesc& k = p.kernels[std::size_t(id - 1)];
      if (k.scope == KernelScope::GlobalAggregation) continue;
      lg.stages.push_back(make_stage(k));
      ops.push_back(k.stencil_op);
      if (k.stencil_op == "iir_temporal") {
        lg.has_iir = true;
        ++n_iir_;
      }
    }
    if (lg.stages.empty()) continue;
    lg.reads_video = first;
    first = false;
    using V = std::vector<std::string>;
    const V chain5 = {"rgba2gray", "iir_temporal", "gaussian", "gradient", "threshold"};
    const V chain4 = {"iir_temporal", "gaussian", "gradient", "threshold"};
    auto radius = [&](std::size_t i) { return lg.stages[i].g_radius; };
    if (lg.reads_video && ops == chain5 && radius(2) >= 1 && radius(2) <= 3)
      lg.kind = LaunchGroup::Chain;
    else if (lg.reads_video && dims_.channels == 1 && ops == chain4 &&
             radius(1) >= 1 && radius(1) <= 3)
      lg.kind = LaunchGroup::Chain;
    else if (lg.reads_video && ops == V{"rgba2gray", "iir_temporal"})
      lg.kind = LaunchGroup::GrayIir;
    else if (ops == V{"gaussian", "gradient", "threshold"})
      lg.kind = LaunchGroup::GaussGradThr;
    else
      lg.kind = LaunchGroup::Stages;
    groups_.push_back(std::move(lg));
  }
  require(!groups_.empty(), ErrorKind::Input, "pipeline has no executable stage");
  const fc_stage& last = groups_.back().stages.back();
  if (last.op == FC_THRESHOLD && is_byte_level(last.white) &&
      is_byte_level(last.black))
    out_type_ = FC_U8;
  for (auto& g : groups_) g.out_type = FC_F32;
  groups_.back().out_type = out_type_;
}

int Executor::converge(const void* video, int in_type, int n_frames, const float* s_true,
                       const float* s_warm, void* stream) {
  require(s_true && s_warm && video, ErrorKind::Input, "converge: null pointer");
  // the stages before the IIR: none (gray video) or one rgba2gray
  std::vector<const fc_stage*> pre;
  const fc_stage* iir = nullptr;
  for (const auto& g : groups_) {
    for (const auto& s : g.stages) {
      if (s.op == FC_IIR_TEMPORAL) {
        iir = &s;
        break;
      }
      pre.push_back(&s);
    }
    if (iir) break;
  }
  require(iir != nullptr && n_iir_ == 1, ErrorKind::Input,
          "converge: the chain needs exactly one IIR stage");
  const bool gray_in = pre.empty();
  require(gray_in ? dims_.channels == 1 : (pre.size() == 1 && pre[0]->op == FC_RGBA2GRAY),
          ErrorKind::Input, "converge: only [rgba2gray,] iir_temporal may open the chain");
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(stream ? stream : own_stream_);
  if (!k_dev_) cuda_check(cudaMalloc(&k_dev_, sizeof(int)), "cudaMalloc(k)");
  cuda_check(fc_iir_converge(gray_in ? nullptr : pre[0], iir, video, in_type, gray_in,
                             fc_dims{dims_.width, dims_.height, n_frames}, s_true, s_warm,
                             k_dev_, st),
             "carry convergence");
  int k = 0;
  cuda_check(cudaMemcpyAsync(&k, k_dev_, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H k");
  cuda_check(cudaStreamSynchronize(st), "converge sync");
  return k;
}

void* Executor::capture(const void* video, int in_type, void* out, void* stream) {
  require(stream != nullptr, ErrorKind::Input, "capture needs a non-default stream");
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  run_device(video, in_type, out, dims_.frames, 0, nullptr, nullptr, st);  // settle lazies
  cuda_check(cudaStreamSynchronize(st), "capture warm-up");
  cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
  try {
    run_device(video, in_type, out, dims_.frames, 0, nullptr, nullptr, st);
  } catch (...) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(st, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  cudaGraph_t g = nullptr;
  cuda_check(cudaStreamEndCapture(st, &g), "end capture");
  cudaGraphExec_t exec = nullptr;
  const cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
  cudaGraphDestroy(g);
  cuda_check(e, "graph instantiate");
  return exec;
}

Executor::~Executor() {
  if (pitched_) cudaFree(pitched_);
  if (k_dev_) cudaFree(k_dev_);
  if (scratch_) cudaFree(scratch_);
  if (stage_) cudaFree(stage_);
  if (s_in_) cudaStreamDestroy(static_cast<cudaStream_t>(s_in_));
  if (s_out_) cudaStreamDestroy(static_cast<cudaStream_t>(s_out_));
  if (own_stream_) cudaStreamDestroy(static_cast<cudaStream_t>(own_stream_));
}

void Executor::ensure_scratch(std::size_t bytes) {
  if (bytes <= scratch_bytes_) return;
  if (scratch_) cuda_check(cudaFree(scratch_), "cudaFree");
  scratch_ = nullptr;
  cuda_check(cudaMalloc(&scratch_, bytes), "cudaMalloc(scratch)");
  scratch_bytes_ = bytes;
}

std::int64_t Executor::launches_per_run() const {
  std::int64_t n = 0;
  for (const auto& g : groups_)
    n += g.kind == LaunchGroup::Stages ? std::int64_t(g.stages.size()) : 1;
  return n;
}

std::string Executor::describe() const {
  std::ostringstream ss;
  ss << "{\"device\": " << device_ << ", \"variant\": " << int(opt_.variant)
     << ", \"output\": \"" << (out_type_ == FC_U8 ? "u8" : "f32")
     << "\", \"launches_per_run\": " << launches_per_run()
     << ", \"last_chain_kernel\": \"" << last_chain_ << "\""
     << ", \"exact_rechecks_total\": " << fc_last_recheck_count();
  // the certified band of an all-fused SPEC chain (gray + IIR + gaussian + threshold)
  for (const auto& g : groups_) {
    if (g.kind != LaunchGroup::Chain || g.stages.size() != 5) continue;
    double c[6];
    if (fc_certified_params(&g.stages[0], &g.stages[1], &g.stages[2], &g.stages[4], c) == 0) {
      ss.precision(17);
      ss << ", \"certified\": {\"g0\": " << c[0] << ", \"g1\": " << c[1]
         << ", \"mlo_n\": " << c[2] << ", \"band_n\": " << c[3] << ", \"S\": " << c[4]
         << ", \"mstar\": " << c[5] << "}";
    }
    break;
  }
  ss << ", \"groups\": [";
  for (std::size_t i = 0; i < groups_.size(); ++i) {
    const auto& g = groups_[i];
    ss << (i ? ", " : "") << "{\"first\": " << g.first << ", \"last\": " << g.last
       << ", \"kernel\": \"" << g.kernel_name() << "\", \"fused\": "
       << (g.kind != LaunchGroup::Stages || g.stages.size() == 1 ? "true" : "false")
       << "}";
  }
  ss << "]}";
  return ss.str();
}

void Executor::run_device(const void* video, int in_type, void* out, int n_frames,
                          int n_warm, const float* state_in, float* state_out,
                          void* stream) {
  require(n_frames >= 0 && n_warm >= 0 && n_warm <= n_frames, ErrorKind::Input,
          "bad frame range");
  require(state_in == nullptr || n_iir_ >= 1, ErrorKind::Input,
          "state_in given but the chain has no IIR stage");
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  fc_set_knobs(&knobs_);
  cudaStream_t st = static_cast<cudaStream_t>(stream ? stream : own_stream_);
  const long long hw = (long long)dims_.width * dims_.height;
  const int C = dims_.channels;
  if (n_iir_ == 0 && n_warm > 0) {  // no recurrence: warm-up frames are moot
    const std::size_t esz = in_type == FC_U8 ? 1 : 4;
    video = static_cast<const char*>(video) + std::size_t(n_warm) * C * hw * esz;
    n_frames -= n_warm;
    n_warm = 0;
  }
  require(n_warm == 0 || n_iir_ == 1, ErrorKind::Input,
          "warm-up ranges need exactly one IIR stage in the chain");
  if (n_frames == 0) return;

  // two f32 ping-pong planes of the largest frame count in flight
  std::size_t plane_bytes =
      (std::size_t(hw) * n_frames * sizeof(float) + 255) & ~std::size_t(255);
  bool need_scratch = in_type == FC_U8 && dims_.channels == 1 &&
                      groups_.front().kind != LaunchGroup::Chain;
  for (const auto& g : groups_)
    if (g.kind == LaunchGroup::Stages || g.kind == LaunchGroup::GrayIir ||
        &g != &groups_.back())
      need_scratch = true;
  if (need_scratch) ensure_scratch(2 * plane_bytes);
  float* buf[2] = {static_cast<float*>(scratch_),
                   scratch_ ? reinterpret_cast<float*>(static_cast<char*>(scratch_) +
                                                       plane_bytes)
                            : nullptr};
  int which = 0;

  const void* cur = video;
  int cur_type = in_type;
  // Upper bound of the values held by `cur` (all >= 0), for the certified
  // F345 kernel's error band; < 0 = unknown (the exact kernel runs instead).
  double cur_max = in_type == FC_U8 ? 255.0 : -1.0;
  int frames = n_frames;   // frames held by `cur`
  int warm = n_warm;       // warm-up frames still at the front of `cur`
  int iir_idx = 0;
  auto state_ptr = [&](const float* base) {
    return base ? base + std::size_t(iir_idx) * hw : nullptr;
  };

  // A single-channel u8 video entering f32 stage kernels is widened first
  // (the streaming chain and rgba2gray read u8 directly).
  if (cur_type == FC_U8 && groups_.front().kind != LaunchGroup::Chain &&
      groups_.front().stages.front().op != FC_RGBA2GRAY) {
    fc_stage conv;
    std::memset(&conv, 0, sizeof conv);
    conv.op = FC_IDENTITY;
    cuda_check(fc_stage_spatial(&conv, cur, FC_U8, buf[which], FC_F32,
                                fc_dims{dims_.width, dims_.height, frames}, st),
               "u8 widen");
    cur = buf[which];
    cur_type = FC_F32;
    which ^= 1;
  }

  for (std::size_t gi = 0; gi < groups_.size(); ++gi) {
    const LaunchGroup& g = groups_[gi];
    bool last_group = gi + 1 == groups_.size();
    void* dst = last_group ? out : buf[which];
    int dst_type = last_group ? out_type_ : FC_F32;
    fc_dims d{dims_.width, dims_.height, frames};
    switch (g.kind) {
      case LaunchGroup::Chain: {
        bool gray_in = g.stages.size() == 4;
        const fc_stage* s = g.stages.data();
        const fc_stage* sgray = gray_in ? nullptr : s;
        const fc_stage* rest = gray_in ? s : s + 1;
        // the frame pipeline's TMA map needs a 16-byte row pitch and base:
        // other widths / bases get planes 0-2 copied into a pitched buffer
        // (one 3-D copy) instead of dropping to the FP64 kernel
        const void* pitched = nullptr;
        int vpitch = 0;
        void* pitched_out = nullptr;
        const int P = (dims_.width + 15) / 16 * 16;
        const bool misaligned = (reinterpret_cast<std::uintptr_t>(cur) & 15) != 0;
        const bool out_misaligned =
            dims_.width % 4 != 0 || (reinterpret_cast<std::uintptr_t>(dst) & 3) != 0;
        // (the certified pipeline, or the exact one: variant "exact" or a chain
        // outside the certified path)
        if (cur_type == FC_U8 && !gray_in && dims_.channels == 4 &&
            (dims_.width % 16 != 0 || misaligned || out_misaligned) &&
            ((opt_.variant != Variant::Exact &&
              fc_chain_pipe_applies(sgray, &rest[0], &rest[1], &rest[3], cur_type, gray_in,
                                    dst_type, d, P)) ||
             fc_chain_pipe2_exact_applies(sgray, &rest[0], &rest[1], &rest[3], cur_type,
                                          gray_in, dst_type, d, P))) {
          const std::size_t vbytes = std::size_t(frames) * 4 * dims_.height * P;
          const std::size_t obytes =
              out_misaligned ? std::size_t(frames - warm) * dims_.height * P : 0;
          const std::size_t need = vbytes + obytes;
          if (need > pitched_bytes_) {
            if (pitched_) cuda_check(cudaFree(pitched_), "cudaFree");
            pitched_ = nullptr;
            cuda_check(cudaMalloc(&pitched_, need), "cudaMalloc(pitched video)");
            pitched_bytes_ = need;
          }
          if (out_misaligned) pitched_out = static_cast<char*>(pitched_) + vbytes;
          cudaMemcpy3DParms cp = {};
          cp.srcPtr = make_cudaPitchedPtr(const_cast<void*>(cur), dims_.width, dims_.width,
                                          4 * dims_.height);
          cp.dstPtr = make_cudaPitchedPtr(pitched_, P, dims_.width, 4 * dims_.height);
          cp.extent = make_cudaExtent(dims_.width, 3 * dims_.height, frames);
          cp.kind = cudaMemcpyDeviceToDevice;
          cuda_check(cudaMemcpy3DAsync(&cp, st), "pitched copy");
          pitched = pitched_;
          vpitch = P;
        }
        cuda_check(fc_fused_chain_pitched(sgray, &rest[0], &rest[1], &rest[2], &rest[3], cur,
                                          pitched, vpitch, pitched_out, P, cur_type, gray_in,
                                          dst, dst_type, d, warm, state_ptr(state_in),
                                          const_cast<float*>(state_ptr(state_out)),
                                          int(opt_.variant), st),
                   "F12345 launch");
        last_chain_ = fc_last_chain_kernel();
        if (pitched) last_chain_ += " on a pitched copy";
        frames -= warm;
        warm = 0;
        ++iir_idx;
        break;
      }
      case LaunchGroup::GrayIir:
        cur_max = stage_range(g.stages[1], stage_range(g.stages[0], cur_max));
        cuda_check(fc_fused_gray_iir(&g.stages[0], &g.stages[1], cur, cur_type,
                                     static_cast<float*>(dst), d, warm,
                                     state_ptr(state_in),
                                     const_cast<float*>(state_ptr(state_out)), st),
                   "F12 launch");
        frames -= warm;
        warm = 0;
        ++iir_idx;
        break;
      case LaunchGroup::GaussGradThr:
        require(cur_type == FC_F32, ErrorKind::Internal, "F345 needs f32 planes");
        cuda_check(fc_fused_gauss_grad_thr_v(&g.stages[0], &g.stages[1], &g.stages[2],
                                             static_cast<const float*>(cur), dst, dst_type, d,
                                             int(opt_.variant), cur_max, st),
                   "F345 launch");
        last_chain_ = fc_last_chain_kernel();
        cur_max = -1.0;
        break;
      case LaunchGroup::Stages:
        for (std::size_t si = 0; si < g.stages.size(); ++si) {
          const fc_stage& s = g.stages[si];
          bool last_stage = si + 1 == g.stages.size();
          void* sdst = (last_stage && last_group) ? out : buf[which];
          int sdst_type = (last_stage && last_group) ? out_type_ : FC_F32;
          fc_dims sd{dims_.width, dims_.height, frames};
          if (s.op == FC_IIR_TEMPORAL) {
            require(cur_type == FC_F32, ErrorKind::Internal, "iir needs f32 planes");
            cuda_check(fc_stage_iir(&s, static_cast<const float*>(cur),
                                    static_cast<float*>(sdst), sd, warm,
                                    state_ptr(state_in),
                                    const_cast<float*>(state_ptr(state_out)), st),
                       "iir launch");
            frames -= warm;
            warm = 0;
            ++iir_idx;
          } else {
            cuda_check(fc_stage_spatial(&s, cur, cur_type, sdst, sdst_type, sd, st),
                       "stage launch");
          }
          cur_max = stage_range(s, cur_max);
          cur = sdst;
          cur_type = sdst_type;
          if (!(last_stage && last_group)) which ^= 1;
        }
        continue;  // cur already advanced
    }
    cur = dst;
    cur_type = dst_type;
    if (!last_group) which ^= 1;
  }
}

void Executor::run_host(const void* video, int in_type, void* out) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  const long long hw = (long long)dims_.width * dims_.height;
  const int C = dims_.channels, F = dims_.frames;
  const std::size_t esz = in_type == FC_U8 ? 1 : 4;
  const std::size_t osz = out_type_ == FC_U8 ? 1 : 4;
  const std::size_t in_frame = std::size_t(C) * hw * esz;
  const std::size_t out_frame = std::size_t(hw) * osz;
  // Channels the chain reads: rgba2gray never touches alpha (simulator.cpp:55),
  // so only planes 0..2 of each frame cross the host link.
  const int read_planes =
      (C == 4 && groups_.front().stages.front().op == FC_RGBA2GRAY) ? 3 : C;

  bool temporal_window = false;
  for (const auto& g : groups_)
    for (const auto& s : g.stages)
      if (s.op == FC_BOX_MEAN && s.rt > 0) temporal_window = true;
  int chunk = opt_.host_chunk_frames;
  if (chunk <= 0)
    chunk = int(std::max<long long>(1, (48LL << 20) / (long long)in_frame));  // ~25 frames at 800x600
  if (temporal_window) chunk = F;  // cannot cut a temporal window
  chunk = std::min(chunk, F);
  const int n_chunks = (F + chunk - 1) / chunk;

  // device staging: 2 video chunks, 2 output chunks, 2 state sets
  auto align = [](std::size_t b) { return (b + 255) & ~std::size_t(255); };
  std::size_t vbytes = align(std::size_t(chunk) * in_frame);
  std::size_t obytes = align(std::size_t(chunk) * out_frame);
  std::size_t sbytes = align(std::size_t(std::max(n_iir_, 1)) * hw * sizeof(float));
  if (2 * (vbytes + obytes + sbytes) > stage_bytes_) {
    if (stage_) cuda_check(cudaFree(stage_), "cudaFree(stage)");
    stage_ = nullptr;
    stage_bytes_ = 0;
    cuda_check(cudaMalloc(&stage_, 2 * (vbytes + obytes + sbytes)), "cudaMalloc(stream)");
    stage_bytes_ = 2 * (vbytes + obytes + sbytes);
  }
  char* mem = static_cast<char*>(stage_);
  char* vb[2] = {mem, mem + vbytes};
  char* ob[2] = {mem + 2 * vbytes, mem + 2 * vbytes + obytes};
  float* sb[2] = {reinterpret_cast<float*>(mem + 2 * (vbytes + obytes)),
                  reinterpret_cast<float*>(mem + 2 * (vbytes + obytes) + sbytes)};
  if (!s_in_) {
    cudaStream_t a, b;
    cuda_check(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking), "stream");
    s_in_ = a;
    s_out_ = b;
  }
  cudaStream_t s_in = static_cast<cudaStream_t>(s_in_), s_out = static_cast<cudaStream_t>(s_out_);
  cudaStream_t s_comp = static_cast<cudaStream_t>(own_stream_);
  std::vector<cudaEvent_t> ev_in(n_chunks), ev_comp(n_chunks), ev_out(n_chunks);
  for (int k = 0; k < n_chunks; ++k) {
    cudaEventCreateWithFlags(&ev_in[k], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_comp[k], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_out[k], cudaEventDisableTiming);
  }
  std::string err;
  try {
    for (int k = 0; k < n_chunks; ++k) {
      int t0 = k * chunk, nf = std::min(chunk, F - t0);
      int b = k & 1;
      // H2D: buffer b is free once chunk k-2's compute has consumed it
      if (k >= 2) cuda_check(cudaStreamWaitEvent(s_in, ev_comp[k - 2], 0), "wait");
      const char* src = static_cast<const char*>(video) + std::size_t(t0) * in_frame;
      if (read_planes == C)
        cuda_check(cudaMemcpyAsync(vb[b], src, std::size_t(nf) * in_frame,
                                   cudaMemcpyHostToDevice, s_in), "H2D");
      else
        cuda_check(cudaMemcpy2DAsync(vb[b], in_frame, src, in_frame,
                                     std::size_t(read_planes) * hw * esz, nf,
                                     cudaMemcpyHostToDevice, s_in), "H2D");
      cuda_check(cudaEventRecord(ev_in[k], s_in), "record");
      // compute: after its input landed and after chunk k-2's D2H freed ob[b]
      cuda_check(cudaStreamWaitEvent(s_comp, ev_in[k], 0), "wait");
      if (k >= 2) cuda_check(cudaStreamWaitEvent(s_comp, ev_out[k - 2], 0), "wait");
      run_device(vb[b], in_type, ob[b], nf, 0, k == 0 || n_iir_ == 0 ? nullptr : sb[b ^ 1],
                 n_iir_ ? sb[b] : nullptr, s_comp);
      cuda_check(cudaEventRecord(ev_comp[k], s_comp), "record");
      // D2H
      cuda_check(cudaStreamWaitEvent(s_out, ev_comp[k], 0), "wait");
      cuda_check(cudaMemcpyAsync(static_cast<char*>(out) + std::size_t(t0) * out_frame,
                                 ob[b], std::size_t(nf) * out_frame,
                                 cudaMemcpyDeviceToHost, s_out), "D2H");
      cuda_check(cudaEventRecord(ev_out[k], s_out), "record");
    }
    cuda_check(cudaStreamSynchronize(s_out), "sync");
    cuda_check(cudaStreamSynchronize(s_comp), "sync");
  } catch (const Error& e) {
    err = e.what();
  }
  cudaStreamSynchronize(s_in);
  cudaStreamSynchronize(s_comp);
  cudaStreamSynchronize(s_out);
  for (int k = 0; k < n_chunks; ++k) {
    cudaEventDestroy(ev_in[k]);
    cudaEventDestroy(ev_comp[k]);
    cudaEventDestroy(ev_out[k]);
  }
  if (!err.empty()) throw Error(ErrorKind::Internal, err);
}

void Executor::run_file(const std::string& in_path, const std::string& out_path) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  std::FILE* fin = std::fopen(in_path.c_str(), "rb");
  require(fin != nullptr, ErrorKind::Input, "cannot open video file: " + in_path);
  std::FILE* fout = nullptr;
  std::unique_ptr<std::FILE, int (*)(std::FILE*)> in_guard(fin, &std::fclose);
  // header: "FPVD", version, width, height, frames, channels, elem type
  unsigned char hdr[28];
  require(std::fread(hdr, 1, 28, fin) == 28 && std::memcmp(hdr, "FPVD", 4) == 0,
          ErrorKind::Input, "not an FPVD video file");
  auto u32 = [&](int i) {
    return std::uint32_t(hdr[i]) | std::uint32_t(hdr[i + 1]) << 8 |
           std::uint32_t(hdr[i + 2]) << 16 | std::uint32_t(hdr[i + 3]) << 24;
  };
  require(u32(4) == 1, ErrorKind::Input, "unsupported FPVD version");
  require(int(u32(8)) == dims_.width && int(u32(12)) == dims_.height &&
              int(u32(16)) == dims_.frames && int(u32(20)) == dims_.channels,
          ErrorKind::Input, "video does not match pipeline dimensions");
  require(u32(24) <= 1, ErrorKind::Input, "unknown FPVD element type");
  const int in_type = u32(24) == 0 ? FC_U8 : FC_F32;

  const long long hw = (long long)dims_.width * dims_.height;
  const int C = dims_.channels, F = dims_.frames;
  const std::size_t esz = in_type == FC_U8 ? 1 : 4;
  const std::size_t osz = out_type_ == FC_U8 ? 1 : 4;
  const std::size_t in_frame = std::size_t(C) * hw * esz, out_frame = std::size_t(hw) * osz;
  const int read_planes =
      (C == 4 && groups_.front().stages.front().op == FC_RGBA2GRAY) ? 3 : C;
  bool temporal_window = false;
  for (const auto& g : groups_)
    for (const auto& st : g.stages)
      if (st.op == FC_BOX_MEAN && st.rt > 0) temporal_window = true;
  int chunk = opt_.host_chunk_frames;
  if (chunk <= 0) chunk = int(std::max<long long>(1, (96LL << 20) / (long long)in_frame));
  if (temporal_window) chunk = F;  // cannot cut a temporal window
  chunk = std::max(1, std::min(chunk, F));
  const int n_chunks = (F + chunk - 1) / chunk;

  fout = std::fopen(out_path.c_str(), "wb");
  require(fout != nullptr, ErrorKind::Input, "cannot write video file: " + out_path);
  std::unique_ptr<std::FILE, int (*)(std::FILE*)> out_guard(fout, &std::fclose);
  {
    unsigned char oh[28];
    std::memcpy(oh, "FPVD", 4);
    const std::uint32_t vals[6] = {1u, std::uint32_t(dims_.width), std::uint32_t(dims_.height),
                                   std::uint32_t(F), 1u, out_type_ == FC_U8 ? 0u : 1u};
    for (int i = 0; i < 6; ++i)
      for (int b = 0; b < 4; ++b) oh[4 + 4 * i + b] = (unsigned char)(vals[i] >> (8 * b));
    require(std::fwrite(oh, 1, 28, fout) == 28, ErrorKind::Input, "write failed: " + out_path);
  }
  if (F == 0) return;

  auto align = [](std::size_t b) { return (b + 255) & ~std::size_t(255); };
  const std::size_t vbytes = align(std::size_t(chunk) * in_frame);
  const std::size_t obytes = align(std::size_t(chunk) * out_frame);
  const std::size_t sbytes = align(std::size_t(std::max(n_iir_, 1)) * hw * sizeof(float));
  char* mem = nullptr;
  char* pin = nullptr;
  cuda_check(cudaMalloc(&mem, 2 * (vbytes + obytes + sbytes)), "cudaMalloc(file stream)");
  if (cudaMallocHost(&pin, 2 * (vbytes + obytes)) != cudaSuccess) {
    cudaFree(mem);
    throw Error(ErrorKind::Internal, "cudaMallocHost(file stream) failed");
  }
  char* vb[2] = {mem, mem + vbytes};
  char* ob[2] = {mem + 2 * vbytes, mem + 2 * vbytes + obytes};
  float* sb[2] = {reinterpret_cast<float*>(mem + 2 * (vbytes + obytes)),
                  reinterpret_cast<float*>(mem + 2 * (vbytes + obytes) + sbytes)};
  char* pi[2] = {pin, pin + vbytes};
  char* po[2] = {pin + 2 * vbytes, pin + 2 * vbytes + obytes};
  if (!s_in_) {
    cudaStream_t a, b;
    cuda_check(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking), "stream");
    s_in_ = a;
    s_out_ = b;
  }
  cudaStream_t s_in = static_cast<cudaStream_t>(s_in_), s_out = static_cast<cudaStream_t>(s_out_);
  cudaStream_t s_comp = static_cast<cudaStream_t>(own_stream_);
  std::vector<cudaEvent_t> ev_in(n_chunks), ev_comp(n_chunks), ev_out(n_chunks);
  for (int k = 0; k < n_chunks; ++k) {
    cudaEventCreateWithFlags(&ev_in[k], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_comp[k], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_out[k], cudaEventDisableTiming);
  }
  auto frames_of = [&](int k) { return std::min(chunk, F - k * chunk); };
  auto write_chunk = [&](int k) {
    cuda_check(cudaEventSynchronize(ev_out[k]), "sync D2H");
    const std::size_t bytes = std::size_t(frames_of(k)) * out_frame;
    require(std::fwrite(po[k & 1], 1, bytes, fout) == bytes, ErrorKind::Input,
            "write failed: " + out_path);
  };
  std::string err;
  ErrorKind kind = ErrorKind::Internal;
  try {
    for (int k = 0; k < n_chunks; ++k) {
      const int nf = frames_of(k), b = k & 1;
      // pinned input b is free once chunk k-2's H2D finished
      if (k >= 2) cuda_check(cudaEventSynchronize(ev_in[k - 2]), "sync H2D");
      const std::size_t bytes = std::size_t(nf) * in_frame;
      require(std::fread(pi[b], 1, bytes, fin) == bytes, ErrorKind::Input,
              "video payload size mismatch");
      if (k >= 2) cuda_check(cudaStreamWaitEvent(s_in, ev_comp[k - 2], 0), "wait");
      if (read_planes == C)
        cuda_check(cudaMemcpyAsync(vb[b], pi[b], bytes, cudaMemcpyHostToDevice, s_in), "H2D");
      else
        cuda_check(cudaMemcpy2DAsync(vb[b], in_frame, pi[b], in_frame,
                                     std::size_t(read_planes) * hw * esz, nf,
                                     cudaMemcpyHostToDevice, s_in),
                   "H2D");
      cuda_check(cudaEventRecord(ev_in[k], s_in), "record");
      cuda_check(cudaStreamWaitEvent(s_comp, ev_in[k], 0), "wait");
      if (k >= 2) cuda_check(cudaStreamWaitEvent(s_comp, ev_out[k - 2], 0), "wait");
      run_device(vb[b], in_type, ob[b], nf, 0, k == 0 || n_iir_ == 0 ? nullptr : sb[b ^ 1],
                 n_iir_ ? sb[b] : nullptr, s_comp);
      cuda_check(cudaEventRecord(ev_comp[k], s_comp), "record");
      cuda_check(cudaStreamWaitEvent(s_out, ev_comp[k], 0), "wait");
      cuda_check(cudaMemcpyAsync(po[b], ob[b], std::size_t(nf) * out_frame,
                                 cudaMemcpyDeviceToHost, s_out),
                 "D2H");
      cuda_check(cudaEventRecord(ev_out[k], s_out), "record");
      // disk write of the previous chunk overlaps this chunk's GPU work
      if (k >= 1) write_chunk(k - 1);
    }
    write_chunk(n_chunks - 1);
  } catch (const Error& e) {
    err = e.what();
    kind = e.kind();
  }
  cudaStreamSynchronize(s_in);
  cudaStreamSynchronize(s_comp);
  cudaStreamSynchronize(s_out);
  for (int k = 0; k < n_chunks; ++k) {
    cudaEventDestroy(ev_in[k]);
    cudaEventDestroy(ev_comp[k]);
    cudaEventDestroy(ev_out[k]);
  }
  cudaFreeHost(pin);  // (the copy streams are the executor's, kept)
  cudaFree(mem);
  if (!err.empty()) throw Error(kind, err);
}

}  // namespace fuseplan
