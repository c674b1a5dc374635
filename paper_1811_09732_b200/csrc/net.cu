// net.cu — the CNN executor over store-lent weights (see nn.hpp).
#include <algorithm>
#include <cmath>
#include <functional>
#include <map>
#include <sstream>

#include "cuda_util.hpp"
#include "nn.hpp"

namespace trims::nn {

struct Net::Step {
  std::function<void(cudaStream_t)> fn;
  uint32_t launches{1};
};

namespace {

struct Act {
  uint16_t* p{nullptr};
  int n{0}, h{1}, w{1}, c{0};
  uint64_t elems() const { return uint64_t(n) * h * w * c; }
};

struct LayerSpec {
  std::string kind;
  std::map<std::string, std::string> kv;
  int i(const char* k, int d = 0) const {
    auto it = kv.find(k);
    return it == kv.end() || it->second.empty() ? d : std::stoi(it->second);
  }
  std::string s(const char* k) const {
    auto it = kv.find(k);
    return it == kv.end() ? std::string() : it->second;
  }
};

std::vector<LayerSpec> parse_arch(const std::string& text) {
  std::vector<LayerSpec> out;
  std::istringstream is(text);
  std::string line;
  while (std::getline(is, line)) {
    std::istringstream ls(line);
    LayerSpec l;
    if (!(ls >> l.kind)) continue;
    std::string tok;
    while (ls >> tok) {
      auto eq = tok.find('=');
      if (eq == std::string::npos) raise(Errc::InvalidArgument, "arch token " + tok);
      l.kv[tok.substr(0, eq)] = tok.substr(eq + 1);
    }
    out.push_back(std::move(l));
  }
  return out;
}

std::string bn_name(const std::string& conv) {
  // torchvision naming: conv1 -> bn1, layerX.Y.convZ -> layerX.Y.bnZ, downsample.0 -> downsample.1
  if (conv.size() > 12 && conv.compare(conv.size() - 12, 12, "downsample.0") == 0)
    return conv.substr(0, conv.size() - 1) + "1";
  std::string b = conv;
  auto pos = b.rfind("conv");
  if (pos == std::string::npos) raise(Errc::InvalidArgument, "no bn name for " + conv);
  b.replace(pos, 4, "bn");
  return b;
}

}  // namespace

uint8_t* Net::alloc(uint64_t bytes) {
  void* p = nullptr;
  TRIMS_CUDA(cudaMalloc(&p, std::max<uint64_t>(bytes, 256)));
  owned_.push_back(p);
  ws_bytes_ += bytes;
  return static_cast<uint8_t*>(p);
}

Net::Net(int device, const std::string& arch, const fmt::Manifest& resident, const uint8_t* weights, int batch)
    : device_(device), batch_(batch) {
  DeviceGuard g(device);
  TRIMS_CUDA(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, device));
  std::map<std::string, const fmt::TensorSpec*> tensors;
  for (const auto& t : resident.tensors) tensors[t.name] = &t;
  auto tensor = [&](const std::string& name, fmt::DType want) -> const uint16_t* {
    auto it = tensors.find(name);
    if (it == tensors.end()) raise(Errc::InvalidArgument, "resident manifest lacks " + name);
    if (it->second->dtype != want) raise(Errc::InvalidArgument, name + " is not resident as bf16");
    return reinterpret_cast<const uint16_t*>(weights + it->second->offset);
  };

  cudaStream_t bind;
  TRIMS_CUDA(cudaStreamCreateWithFlags(&bind, cudaStreamNonBlocking));
  const std::vector<LayerSpec> layers = parse_arch(arch);
  int last_fc = -1;
  for (size_t i = 0; i < layers.size(); ++i)
    if (layers[i].kind == "fc") last_fc = int(i);

  std::map<std::string, Act> named;
  Act cur;
  uint16_t* col = nullptr;  // shared im2col scratch
  uint64_t col_elems = 0;
  // First pass sizes the im2col scratch; steps keep a pointer to `col` slot.
  std::vector<std::function<void()>> fixups;
  auto conv_shape = [&](const Act& in, const LayerSpec& l, int& P, int& Q) {
    const int k = l.i("k", 1), st = l.i("stride", 1), pad = l.i("pad", 0);
    P = (in.h + 2 * pad - k) / st + 1;
    Q = (in.w + 2 * pad - k) / st + 1;
  };
  {
    // size pass
    Act a;
    for (const auto& l : layers) {
      if (l.kind == "input") {
        a = {nullptr, batch, l.i("hw"), l.i("hw"), l.i("c", 3)};
      } else if (l.kind == "conv") {
        Act in = l.s("src").empty() ? a : named[l.s("src")];
        int P, Q;
        conv_shape(in, l, P, Q);
        const int k = l.i("k", 1), groups = l.i("groups", 1), cg = l.i("cin") / groups;
        const bool direct = k == 1 && l.i("stride", 1) == 1 && l.i("pad", 0) == 0 && groups == 1;
        if (!direct) {
          const uint64_t kp = (uint64_t(k) * k * cg + 7) / 8 * 8;
          col_elems = std::max<uint64_t>(col_elems, uint64_t(batch) * P * Q * kp);
        }
        Act o{nullptr, batch, P, Q, l.i("cout")};
        if (!l.s("out").empty()) named[l.s("out")] = o;
        a = o;
      } else if (l.kind == "pool_max") {
        const int k = l.i("k"), st = l.i("stride", k), pad = l.i("pad", 0);
        a = {nullptr, batch, (a.h + 2 * pad - k) / st + 1, (a.w + 2 * pad - k) / st + 1, a.c};
        if (!l.s("out").empty()) named[l.s("out")] = a;
      } else if (l.kind == "pool_avg") {
        a = {nullptr, batch, 1, 1, a.c};
      } else if (l.kind == "flatten") {
        a = {nullptr, batch, 1, 1, a.h * a.w * a.c};
      } else if (l.kind == "fc") {
        a = {nullptr, batch, 1, 1, l.i("cout")};
      }
    }
    named.clear();
  }
  if (col_elems) col = reinterpret_cast<uint16_t*>(alloc(col_elems * 2));

  for (size_t li = 0; li < layers.size(); ++li) {
    const LayerSpec& l = layers[li];
    if (l.kind == "input") {
      in_hw_ = l.i("hw");
      in_c_ = l.i("c", 3);
      input_ = reinterpret_cast<float*>(alloc(uint64_t(batch) * in_c_ * in_hw_ * in_hw_ * 4));
      cur = {reinterpret_cast<uint16_t*>(alloc(uint64_t(batch) * in_c_ * in_hw_ * in_hw_ * 2)), batch, in_hw_, in_hw_,
             in_c_};
      const float* in = input_;
      Act o = cur;
      const int C = in_c_, HW = in_hw_;
      steps_.push_back(std::make_unique<Step>(
          Step{[=](cudaStream_t s) { input_prep(in, o.p, o.n, C, HW, HW, s); }, 1}));
    } else if (l.kind == "conv") {
      const Act in = l.s("src").empty() ? cur : named.at(l.s("src"));
      int P, Q;
      conv_shape(in, l, P, Q);
      const int k = l.i("k", 1), st = l.i("stride", 1), pad = l.i("pad", 0), groups = l.i("groups", 1);
      const int cin = l.i("cin"), cout = l.i("cout"), cg = cin / groups, kg = cout / groups;
      if (in.c != cin) raise(Errc::InvalidArgument, l.s("name") + ": input channels mismatch");
      const uint64_t M = uint64_t(batch) * P * Q;
      const int rsc = k * k * cg, kp = (rsc + 7) / 8 * 8;
      const std::string name = l.s("name");
      const uint16_t* W = tensor(name + ".weight", fmt::DType::BF16);
      if (kp != rsc) {  // TMA rows must be 16-byte multiples: private zero-padded copy
        auto* wp = reinterpret_cast<uint16_t*>(alloc(uint64_t(cout) * kp * 2));
        pad_rows(W, cout, rsc, wp, kp, bind);
        W = wp;
      }
      float* scale = nullptr;
      float* bias = nullptr;
      if (l.i("bn")) {
        const std::string bn = bn_name(name);
        scale = reinterpret_cast<float*>(alloc(uint64_t(cout) * 4));
        bias = reinterpret_cast<float*>(alloc(uint64_t(cout) * 4));
        nn::bn_fold(tensor(bn + ".weight", fmt::DType::BF16), tensor(bn + ".bias", fmt::DType::BF16),
                    tensor(bn + ".running_mean", fmt::DType::BF16), tensor(bn + ".running_var", fmt::DType::BF16),
                    1e-5f, cout, scale, bias, bind);
      } else if (l.i("bias")) {
        bias = reinterpret_cast<float*>(alloc(uint64_t(cout) * 4));
        bf16_to_f32(tensor(name + ".bias", fmt::DType::BF16), bias, cout, bind);
      }
      const uint16_t* res = nullptr;
      if (!l.s("res").empty()) {
        const Act& r = named.at(l.s("res"));
        if (r.elems() != M * cout) raise(Errc::InvalidArgument, name + ": residual shape mismatch");
        res = r.p;
      }
      Act out{reinterpret_cast<uint16_t*>(alloc(M * cout * 2)), batch, P, Q, cout};
      const bool direct = k == 1 && st == 1 && pad == 0 && groups == 1;
      for (int gi = 0; gi < groups; ++gi) {
        const uint16_t* A = direct ? in.p : col;
        if (!direct) {
          Act src = in;
          steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) {
            nn::im2col(src.p, col, src.n, src.h, src.w, src.c, gi * cg, cg, k, k, st, pad, P, Q, kp, s);
          }, 1}));
        }
        gemm::Epilogue e{out.p + uint64_t(gi) * kg, uint64_t(cout), scale ? scale + gi * kg : nullptr,
                         bias ? bias + gi * kg : nullptr, res ? res + uint64_t(gi) * kg : nullptr, uint64_t(cout),
                         l.i("relu") != 0};
        gemm::Prepared prep = gemm::prepare({A, M, uint64_t(kp), uint64_t(direct ? cin : kp)},
                                            {W + uint64_t(gi) * kg * kp, uint64_t(kg), uint64_t(kp), uint64_t(kp)}, e);
        steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) { gemm::run(prep, s); }, 1}));
      }
      flops_ += 2.0 * double(M) * cout * rsc;
      if (!l.s("out").empty()) named[l.s("out")] = out;
      cur = out;
    } else if (l.kind == "pool_max") {
      const int k = l.i("k"), st = l.i("stride", k), pad = l.i("pad", 0);
      const Act in = cur;
      const int P = (in.h + 2 * pad - k) / st + 1, Q = (in.w + 2 * pad - k) / st + 1;
      Act out{reinterpret_cast<uint16_t*>(alloc(uint64_t(batch) * P * Q * in.c * 2)), batch, P, Q, in.c};
      steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) {
        nn::maxpool(in.p, out.p, in.n, in.h, in.w, in.c, k, st, pad, P, Q, s);
      }, 1}));
      if (!l.s("out").empty()) named[l.s("out")] = out;
      cur = out;
    } else if (l.kind == "pool_avg") {
      const Act in = cur;
      Act out{reinterpret_cast<uint16_t*>(alloc(uint64_t(batch) * in.c * 2)), batch, 1, 1, in.c};
      steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) {
        nn::avgpool_global(in.p, out.p, in.n, in.h * in.w, in.c, s);
      }, 1}));
      cur = out;
    } else if (l.kind == "flatten") {
      const Act in = cur;
      if (in.h * in.w > 1) {  // FC weights expect torch's NCHW flatten order
        Act out{reinterpret_cast<uint16_t*>(alloc(in.elems() * 2)), batch, 1, 1, in.h * in.w * in.c};
        steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) {
          nn::flatten_nchw(in.p, out.p, in.n, in.h * in.w, in.c, s);
        }, 1}));
        cur = out;
      } else {
        cur = {in.p, batch, 1, 1, in.c};
      }
    } else if (l.kind == "fc") {
      const Act in = cur;
      const int cin = l.i("cin"), cout = l.i("cout");
      if (in.c != cin) raise(Errc::InvalidArgument, l.s("name") + ": fc input mismatch");
      const uint16_t* W = tensor(l.s("name") + ".weight", fmt::DType::BF16);
      float* bias = nullptr;
      if (l.i("bias")) {
        bias = reinterpret_cast<float*>(alloc(uint64_t(cout) * 4));
        bf16_to_f32(tensor(l.s("name") + ".bias", fmt::DType::BF16), bias, cout, bind);
      }
      const bool last = int(li) == last_fc;
      const bool relu = l.i("relu") != 0;
      Act out{reinterpret_cast<uint16_t*>(alloc(uint64_t(batch) * cout * 2)), batch, 1, 1, cout};
      if (last) {
        classes_ = cout;
        logits_ = reinterpret_cast<float*>(alloc(uint64_t(batch) * cout * 4));
      }
      float* lg = last ? logits_ : nullptr;
      const int sms = sms_;
      if (batch <= 8) {  // HBM-bound GEMV: weights streamed once
        steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) {
          nn::gemv(in.p, batch, cin, W, cout, bias, relu, out.p, lg, cout, sms, s);
        }, 1}));
      } else {
        gemm::Epilogue e{out.p, uint64_t(cout), nullptr, bias, nullptr, 0, relu};
        gemm::Prepared prep = gemm::prepare({in.p, uint64_t(batch), uint64_t(cin), uint64_t(cin)},
                                            {W, uint64_t(cout), uint64_t(cin), uint64_t(cin)}, e);
        steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) { gemm::run(prep, s); }, 1}));
        if (last) {
          const int n = batch * cout;
          steps_.push_back(
              std::make_unique<Step>(Step{[=](cudaStream_t s) { nn::bf16_to_f32(out.p, lg, n, s); }, 1}));
        }
      }
      flops_ += 2.0 * double(batch) * cin * cout;
      cur = out;
    } else {
      raise(Errc::InvalidArgument, "unknown layer kind " + l.kind);
    }
  }
  if (!logits_) raise(Errc::InvalidArgument, "architecture has no fc output");
  for (const auto& s : steps_) launches_ += s->launches;
  TRIMS_CUDA(cudaStreamSynchronize(bind));
  cudaStreamDestroy(bind);
  TRIMS_CUDA(cudaStreamCreateWithFlags(&capture_stream_, cudaStreamNonBlocking));
}

Net::~Net() {
  DeviceGuard g(device_, /*nothrow=*/true);
  if (exec_) cudaGraphExecDestroy(exec_);
  if (graph_) cudaGraphDestroy(graph_);
  if (capture_stream_) cudaStreamDestroy(capture_stream_);
  for (void* p : owned_) cudaFree(p);
}

void Net::record(cudaStream_t stream) {
  for (const auto& s : steps_) s->fn(stream);
}

void Net::run(cudaStream_t stream, bool use_graph) {
  DeviceGuard g(device_);
  if (!use_graph) {
    record(stream);
    return;
  }
  if (!exec_) {
    TRIMS_CUDA(cudaStreamBeginCapture(capture_stream_, cudaStreamCaptureModeThreadLocal));
    record(capture_stream_);
    TRIMS_CUDA(cudaStreamEndCapture(capture_stream_, &graph_));
    TRIMS_CUDA(cudaGraphInstantiate(&exec_, graph_, 0));
  }
  TRIMS_CUDA(cudaGraphLaunch(exec_, stream));
}

}  // namespace trims::nn
