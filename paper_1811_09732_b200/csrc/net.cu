// net.cu — the CNN executor over store-lent weights (see nn.hpp).
//
// Construction ("bind") sizes and allocates the private workspace once and
// records every layer as a step. Everything that depends on WHERE the shared
// weights live (B-operand tensor maps, GEMV weight pointers, folded BN
// scale/shift, fp32 biases, zero-padded conv1 filters) is recomputed by
// rebind() from resident-manifest offsets, so a client keeps its executor
// across store evictions/reloads and only pays a few microseconds per layer
// when a new generation of the model is published.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <functional>
#include <map>
#include <optional>
#include <sstream>

#include "cuda_util.hpp"
#include "nn.hpp"

namespace trims::nn {

struct Net::Step {
  std::function<void(cudaStream_t)> run;
  std::function<void(cudaStream_t)> rebind;  // weight-dependent state (may be empty)
  uint32_t launches{1};
  int branch{-1};  // >= 0: runs on the side stream as independent branch #branch
  std::vector<int> joins;  // branches whose output this step reads: wait for them first
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

// TRIMS_IMPLICIT_CONV=0 goes back to im2col + GEMM (A/B switch).
bool implicit_enabled();

// The first conv builds its columns from the fp32 input directly when it
// would im2col anyway (not 1x1/stride 1, not implicit, one group).
bool first_conv_fusable(const LayerSpec& l) {
  const int k = l.i("k", 1), groups = l.i("groups", 1);
  const bool direct = k == 1 && l.i("stride", 1) == 1 && l.i("pad", 0) == 0 && groups == 1;
  const bool implicit = !direct && (l.i("cin") / groups) % 64 == 0 && implicit_enabled();
  return !direct && !implicit && groups == 1 && k * k * l.i("cin") <= 504;  // im2col_input: Kp <= 512
}

bool implicit_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TRIMS_IMPLICIT_CONV");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

// TRIMS_BRANCHES=1 runs independent branches on a side stream. Off by
// default: the fork/join edges cost ResNet-50 more than the overlap gains
// (0.336 vs 0.315 ms per forward, profiles/r02a_forward_ab.log), because the
// shortcut GEMM then waits for its producer's full completion instead of a
// programmatic edge.
bool branches_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TRIMS_BRANCHES");
    return e && std::string(e) == "1";
  }();
  return on;
}

// TRIMS_GROUP_PAIR=0: the two groups of a 2-group conv launch separately
// (A/B switch; on: one paired GEMM launch, and one im2col for both groups).
bool group_pair_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TRIMS_GROUP_PAIR");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

// TRIMS_PAIR=0 launches ResNet's downsample and the stage's first 1x1 conv
// (same input, independent) separately instead of as one grouped launch.
bool pairing_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TRIMS_PAIR");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

// TRIMS_TILE_PICK=rule keeps the older tile-width / split rules instead of
// gemm::choose_tiles' cost model (A/B switch).
bool tile_model_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TRIMS_TILE_PICK");
    return !(e && std::string(e) == "rule");
  }();
  return on;
}

// TRIMS_TP_WIDE=0: throughput / lean executors keep the latency rule's tile
// widths instead of the widest tiles (A/B switch).
bool tp_wide_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TRIMS_TP_WIDE");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

// TRIMS_PERSIST: 0 = no persistent GEMMs, 1 = for multi-wave layers except
// long-k-loop 2-SM pairs, 2 = every multi-wave layer launched alone (default:
// VGG-16 b32 2.166 -> 1.624 ms, ResNet-50 b32 1.176 -> 1.043, VGG-16 b1
// 0.2125 -> 0.2048; mode 1 within 1 %; profiles/r3/persist_ab.log).
int persist_mode() {
  static const int m = [] {
    const char* e = std::getenv("TRIMS_PERSIST");
    return e ? std::atoi(e) : 2;
  }();
  return m;
}

// TRIMS_POOL_FUSE=0: 2x2 max pools stay separate launches (A/B switch).
bool pool_fuse_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TRIMS_POOL_FUSE");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

// TRIMS_SPLITK=0 turns split-K off (A/B switch).
bool splitk_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TRIMS_SPLITK");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

}  // namespace

uint8_t* Net::alloc(uint64_t bytes) {
  void* p = nullptr;
  TRIMS_CUDA(cudaMalloc(&p, std::max<uint64_t>(bytes, 256)));
  owned_.push_back(p);
  ws_bytes_ += bytes;
  return static_cast<uint8_t*>(p);
}

Net::Net(int device, const std::string& arch, const fmt::Manifest& resident, const uint8_t* weights, int batch,
         int flags)
    : device_(device), batch_(batch) {
  // Latency mode (default) splits K over more CTAs to cut one request's
  // latency; throughput mode keeps one CTA per output tile, so concurrent
  // clients' kernels pack the SMs (16 MPS clients on ResNet-50: 12.0k vs 5.9k
  // requests/s, profiles/r3/mps_mode_ab.log).
  const bool split_ok = splitk_enabled() && !(flags & (kNetThroughput | kNetLean));
  const bool lean = (flags & kNetLean) != 0;
  DeviceGuard g(device);
  TRIMS_CUDA(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, device));
  std::map<std::string, const fmt::TensorSpec*> tensors;
  for (const auto& t : resident.tensors) tensors[t.name] = &t;
  // Weights are addressed as offsets into the resident blob; `wbase_` is the
  // current generation's base (set by rebind()).
  auto offset_of = [&](const std::string& name) -> uint64_t {
    auto it = tensors.find(name);
    if (it == tensors.end()) raise(Errc::InvalidArgument, "resident manifest lacks " + name);
    if (it->second->dtype != fmt::DType::BF16) raise(Errc::InvalidArgument, name + " is not resident as bf16");
    return it->second->offset;
  };
  const uint8_t* const* wb = &wbase_;
  auto wptr = [wb](uint64_t off) { return reinterpret_cast<const uint16_t*>(*wb + off); };

  const std::vector<LayerSpec> layers = parse_arch(arch);
  int last_fc = -1;
  for (size_t i = 0; i < layers.size(); ++i)
    if (layers[i].kind == "fc") last_fc = int(i);

  auto conv_shape = [&](const Act& in, const LayerSpec& l, int& P, int& Q) {
    const int k = l.i("k", 1), st = l.i("stride", 1), pad = l.i("pad", 0);
    P = (in.h + 2 * pad - k) / st + 1;
    Q = (in.w + 2 * pad - k) / st + 1;
  };
  std::map<std::string, Act> named;
  uint64_t col_elems = 0;
  {  // size pass: the shared im2col scratch
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
        const bool implicit = !direct && cg % 64 == 0 && implicit_enabled();
        if (!direct && !implicit)  // a 2-group conv keeps both groups' columns (one im2col, one paired GEMM launch)
          col_elems = std::max<uint64_t>(col_elems, uint64_t(groups == 2 ? 2 : 1) * batch * P * Q *
                                                        ((uint64_t(k) * k * cg + 7) / 8 * 8));
        a = {nullptr, batch, P, Q, l.i("cout")};
        if (!l.s("out").empty()) named[l.s("out")] = a;
      } else if (l.kind == "pool_max") {
        const int k = l.i("k"), st = l.i("stride", k), pad = l.i("pad", 0);
        a = {nullptr, batch, (a.h + 2 * pad - k) / st + 1, (a.w + 2 * pad - k) / st + 1, a.c};
        if (!l.s("out").empty()) named[l.s("out")] = a;
      } else if (l.kind == "pool_avg") {
        a = {nullptr, batch, 1, 1, a.c};
      } else if (l.kind == "flatten") {
        a = {nullptr, batch, 1, 1, a.h * a.w * a.c};
      }
    }
    named.clear();
  }
  uint16_t* col = col_elems ? reinterpret_cast<uint16_t*>(alloc(col_elems * 2)) : nullptr;
  Act cur;

  std::map<std::string, int> branch_of;  // named output -> side branch producing it
  bool flat_done = false;                // a pool wrote its output flattened (NCHW) for the next flatten
  // A GEMM held back to share the next layer's launch (an independent conv
  // reading the same input): its prepared GEMM and rebind.
  struct Pending {
    std::shared_ptr<gemm::Prepared> prep;
    std::function<void(cudaStream_t)> rebind;
  };
  std::optional<Pending> pending;
  bool pool_fused = false;  // the previous conv wrote this pool layer's output
  for (size_t li = 0; li < layers.size(); ++li) {
    const LayerSpec& l = layers[li];
    if (pool_fused) {
      pool_fused = false;
      taps_.push_back({cur.p, cur.n, cur.h, cur.w, cur.c, 0});
      continue;
    }
    const size_t first_step = steps_.size();
    Act produced;  // this layer's output buffer (the parity tap)
    std::vector<int> joins;
    for (const char* ref : {"src", "res"}) {
      auto it = branch_of.find(l.s(ref));
      if (it != branch_of.end()) {
        joins.push_back(it->second);
        branch_of.erase(it);
      }
    }
    auto attach_joins = [&] {
      if (!joins.empty() && steps_.size() > first_step) steps_[first_step]->joins = joins;
    };
    if (l.kind == "input") {
      in_hw_ = l.i("hw");
      in_c_ = l.i("c", 3);
      input_ = reinterpret_cast<float*>(alloc(uint64_t(batch) * in_c_ * in_hw_ * in_hw_ * 4));
      cur = {reinterpret_cast<uint16_t*>(alloc(uint64_t(batch) * in_c_ * in_hw_ * in_hw_ * 2)), batch, in_hw_, in_hw_,
             in_c_};
      const float* in = input_;
      const Act o = cur;
      const int C = in_c_, HW = in_hw_;
      // A first conv that im2cols the input reads the fp32 NCHW input itself
      // (im2col_input); otherwise the input is converted to NHWC bf16 here.
      const bool fused = li + 1 < layers.size() && layers[li + 1].kind == "conv" && layers[li + 1].s("src").empty() &&
                         first_conv_fusable(layers[li + 1]);
      if (!fused)
        steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) { input_prep(in, o.p, o.n, C, HW, HW, s); }}));
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
      const uint64_t w_off = offset_of(name + ".weight");
      // TMA rows must be 16-byte multiples: conv1-like filters get a private zero-padded copy
      uint16_t* wpad = kp != rsc ? reinterpret_cast<uint16_t*>(alloc(uint64_t(cout) * kp * 2)) : nullptr;
      float* scale = nullptr;
      float* bias = nullptr;
      std::function<void(cudaStream_t)> bind_params;
      if (l.i("bn")) {
        const std::string bn = bn_name(name);
        scale = reinterpret_cast<float*>(alloc(uint64_t(cout) * 4));
        bias = reinterpret_cast<float*>(alloc(uint64_t(cout) * 4));
        const uint64_t og = offset_of(bn + ".weight"), ob = offset_of(bn + ".bias"),
                       om = offset_of(bn + ".running_mean"), ov = offset_of(bn + ".running_var");
        folds_.push_back({og, ob, om, ov, scale, bias, cout});  // folded in one batched launch per rebind
      } else if (l.i("bias")) {
        bias = reinterpret_cast<float*>(alloc(uint64_t(cout) * 4));
        const uint64_t ob = offset_of(name + ".bias");
        bind_params = [=](cudaStream_t s) { bf16_to_f32(wptr(ob), bias, cout, s); };
      }
      const uint16_t* res = nullptr;
      if (!l.s("res").empty()) {
        const Act& r = named.at(l.s("res"));
        if (r.elems() != M * cout) raise(Errc::InvalidArgument, name + ": residual shape mismatch");
        res = r.p;
      }
      Act out{reinterpret_cast<uint16_t*>(alloc(M * cout * 2)), batch, P, Q, cout};
      const bool direct = k == 1 && st == 1 && pad == 0 && groups == 1;
      // Implicit GEMM (A read from the NHWC activation by 4-D TMA, no im2col
      // pass) whenever the channels tile by 64.
      // Grouped convs go implicit per group when a group's channels tile by 64.
      const bool implicit = !direct && cg % 64 == 0 && implicit_enabled();
      // A conv whose output only feeds a later layer by name (the next layer
      // reads its own `src`, e.g. ResNet's downsample shortcut) is an
      // independent branch: it runs on a side stream concurrently with the
      // main path and is joined by the first layer that references it.
      const bool branch = branches_enabled() && groups == 1 && (direct || implicit) && !l.s("out").empty() &&
                          li + 1 < layers.size() && !layers[li + 1].s("src").empty();
      // A 2x2 / 2 max pool right after this conv runs in the GEMM's epilogue
      // (one dependent launch less; VGG): on the staged tile, or on each
      // split-K owner's reduced slice. Not before a flatten: that pool writes
      // NCHW itself.
      const LayerSpec* nx = li + 1 < layers.size() ? &layers[li + 1] : nullptr;
      const bool pool_cand = pool_fuse_enabled() && implicit && groups == 1 && !branch && l.s("out").empty() &&
                             l.s("res").empty() && nx && nx->kind == "pool_max" && nx->i("k") == 2 &&
                             nx->i("stride", 2) == 2 && nx->i("pad", 0) == 0 && nx->s("out").empty() &&
                             nx->s("src").empty() && P % 2 == 0 && Q % 2 == 0;
      // ... before a flatten only on a split-K launch (its owners store the
      // pooled slice NCHW, torch's flatten order, with thread stores)
      const bool pool_flat = li + 2 < layers.size() && layers[li + 2].kind == "flatten" && P * Q > 4;
      // Off by default: the NCHW thread stores made VGG-16 b1 slower than the
      // separate pool (0.1885 -> 0.1933 ms, profiles/r3/pool_box_flat_ab.log).
      static const bool flat_fuse = [] {  // A/B: TRIMS_POOL_FLAT=1 fuses it
        const char* e = std::getenv("TRIMS_POOL_FLAT");
        return e && std::string(e) == "1";
      }();
      // tile box for a fused pool: taller boxes for a single-wave layer
      // (VGG-16 b1 0.1885 -> 0.1862 ms), least padding for multi-wave ones
      // (b32 1.483 -> 1.399)
      // TRIMS_AVG_FUSE=0: the global average pool stays a separate launch (A/B)
      static const bool avg_fuse = [] {
        const char* e = std::getenv("TRIMS_AVG_FUSE");
        return !(e && std::string(e) == "0");
      }();
      // (a named output is fine when no later layer reads it: ResNet's last
      // block names its output for a residual nobody takes)
      const bool out_unread = [&] {
        const std::string o = l.s("out");
        for (size_t j = li + 1; !o.empty() && j < layers.size(); ++j)
          if (layers[j].s("src") == o || layers[j].s("res") == o) return false;
        return true;
      }();
      const bool avg_cand = avg_fuse && (implicit || direct) && groups == 1 && !branch && out_unread && nx &&
                            nx->kind == "pool_avg" && nx->s("out").empty() && nx->s("src").empty();
      const int pool_box = !pool_cand ? 0 : uint64_t(batch) * P * Q <= uint64_t(sms_) * 128 ? 2 : 1;
      bool fused_here = false;
      Act pout{};
      bool first_group = true;
      // both groups of a 2-group im2col conv (AlexNet conv2): one im2col launch
      // into side-by-side column buffers, then one paired GEMM launch
      const bool gcol = group_pair_enabled() && groups == 2 && !direct && !implicit &&
                        !(li == 1 && layers[0].kind == "input" && l.s("src").empty() && first_conv_fusable(l));
      for (int gi = 0; gi < groups; ++gi) {
        const uint16_t* A = direct ? in.p : gcol ? col + uint64_t(gi) * M * kp : col;
        if (gcol) {
          if (gi == 0) {
            const Act src = in;
            steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) {
              nn::im2col(src.p, col, src.n, src.h, src.w, src.c, 0, cg, k, k, st, pad, P, Q, kp, s, 2);
            }}));
          }
        } else if (!direct && !implicit) {
          const Act src = in;
          if (li == 1 && layers[0].kind == "input" && l.s("src").empty() && first_conv_fusable(l)) {
            const float* x = input_;
            steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) {
              nn::im2col_input(x, col, src.n, src.c, src.h, src.w, k, k, st, pad, P, Q, kp, s);
            }}));
          } else {
            steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) {
              nn::im2col(src.p, col, src.n, src.h, src.w, src.c, gi * cg, cg, k, k, st, pad, P, Q, kp, s);
            }}));
          }
        }
        gemm::Epilogue e{out.p + uint64_t(gi) * kg, uint64_t(cout), scale ? scale + gi * kg : nullptr,
                         bias ? bias + gi * kg : nullptr, res ? res + uint64_t(gi) * kg : nullptr, uint64_t(cout),
                         l.i("relu") != 0};
        // A-side map and tile width are fixed; the B map follows the weights.
        const gemm::Operand Bop{wpad ? wpad : reinterpret_cast<const uint16_t*>(uintptr_t(256)), uint64_t(kg),
                                uint64_t(kp), uint64_t(kp)};
        auto prep = std::make_shared<gemm::Prepared>(
            implicit ? gemm::prepare_conv(
                           in.p, gemm::conv_geom(batch, in.h, in.w, cin, k, k, st, pad, P, Q, cg, gi * cg, pool_box),
                           Bop, e)
                     : gemm::prepare({A, M, uint64_t(kp), uint64_t(direct ? cin : kp)}, Bop, e));
        // the same GEMM prepared with another tile width
        auto remake = [&](int bn) {
          return std::make_shared<gemm::Prepared>(
              implicit ? gemm::prepare_conv(
                             in.p, gemm::conv_geom(batch, in.h, in.w, cin, k, k, st, pad, P, Q, cg, gi * cg, pool_box),
                             Bop, e, bn)
                       : gemm::prepare({A, M, uint64_t(kp), uint64_t(direct ? cin : kp)}, Bop, e, bn));
        };
        if (split_ok && tile_model_enabled()) {
          int bn = 0, sp = 1;
          bool pr = false;
          gemm::choose_tiles(gemm::tile_rows(*prep), uint64_t(kg), uint64_t(kp), sms_, &bn, &sp, &pr);
          if (bn != prep->bn) prep = remake(bn);
          prep->splits = sp;
          prep->pair = pr;
        } else if (split_ok) {
          prep->splits = gemm::pick_splits(gemm::tile_rows(*prep), uint64_t(kg), uint64_t(kp), prep->bn, sms_);
        } else if (!split_ok && (flags & (kNetThroughput | kNetLean))) {
          // Many clients share the GPU: wider tiles, fewer CTAs (each CTA's
          // fixed cost is paid once per 128 instead of 64 output channels).
          // 16 MPS clients on ResNet-50: 14.1k -> 15.6k req/s
          // (profiles/r3/mps_bn_ab.log). Lean has no 256-wide variant.
          const int want = (!lean && kg >= 256 && kg % 256 == 0) ? 256 : kg >= 128 ? 128 : 64;
          if (tp_wide_enabled() && want != prep->bn) prep = remake(want);
        }
        // second GEMM of a grouped launch: the first one's tile width
        if (pending && groups == 1 && pending->prep->bn != prep->bn &&
            !(pending->prep->bn == 256 && prep->N % 256)) {
          const int sp = prep->splits;
          prep = remake(pending->prep->bn);
          prep->splits = pending->prep->bn == 256 ? 1 : sp;
        }
        prep->lean = lean;
        // Pair with the next layer when it is an independent conv on the same
        // input (ResNet: downsample + the stage's first 1x1 conv).
        const bool pair_first = pairing_enabled() && !branches_enabled() && groups == 1 && !l.s("src").empty() &&
                                li + 1 < layers.size() && layers[li + 1].kind == "conv" &&
                                layers[li + 1].s("src") == l.s("src") && layers[li + 1].i("groups", 1) == 1 &&
                                !pending;
        const bool pair_second = pending && groups == 1;
        // The two groups of a 2-group implicit conv (AlexNet conv4/conv5) are
        // independent GEMMs on disjoint input channels and output columns: one
        // launch runs both (TRIMS_GROUP_PAIR=0: A/B).
        const bool gpair_first =
            group_pair_enabled() && groups == 2 && (implicit || gcol) && gi == 0 && !pending && !pool_cand && !avg_cand;
        const bool gpair_second = groups == 2 && (implicit || gcol) && gi == 1 && bool(pending);
        if (pair_first || pair_second || gpair_first || gpair_second) prep->pair = false;  // grouped launches run single-CTA GEMMs
        // weight multicast across M-tiles for a GEMM launched alone (latency mode)
        if (split_ok && !pair_first && !pair_second && !gpair_first && !gpair_second) prep->mc = gemm::pick_mc(*prep, sms_);
        // a multi-wave GEMM launched alone runs persistent CTAs (one per SM,
        // double-buffered accumulators: each tile's epilogue overlaps the next
        // tile's k-loop), in place of a 2-SM pair too (mode 1: only when the
        // pair's k-loop is short)
        if (!pair_first && !pair_second && !gpair_first && !gpair_second && !lean && prep->splits == 1 && prep->mc <= 1 &&
            prep->tma_out) {
          const uint64_t tiles = gemm::tile_rows(*prep) / 128 * ((prep->N + prep->bn - 1) / prep->bn);
          const uint64_t kb = (uint64_t(kp) + 63) / 64;
          const int mode = persist_mode();
          if (mode && tiles > uint64_t(sms_) && (!prep->pair || mode == 2 || kb <= 8)) {
            prep->pair = false;
            prep->persist = true;
          }
        }
        if (pool_cand && !pair_first && !pair_second && !prep->pair && prep->mc <= 1 && prep->tma_out &&
            (!pool_flat || (prep->splits > 1 && flat_fuse))) {
          pout = {reinterpret_cast<uint16_t*>(alloc(uint64_t(batch) * (P / 2) * (Q / 2) * cout * 2)), batch, P / 2,
                  Q / 2, cout};
          gemm::ConvGeom g = gemm::conv_geom(batch, in.h, in.w, cin, k, k, st, pad, P, Q, cg, gi * cg, pool_box);
          g.pool = pool_flat ? 2 : 1;
          gemm::Epilogue ep = e;
          ep.out = pout.p;
          auto np = std::make_shared<gemm::Prepared>(gemm::prepare_conv(in.p, g, Bop, ep, prep->bn));
          np->persist = prep->persist;
          np->lean = prep->lean;
          np->splits = prep->splits;
          prep = np;
          fused_here = true;
        }
        // A global average pool right after the last conv (ResNet) runs in
        // that GEMM's split-K owners: each tile is one whole image, so an owner
        // holds every pixel of its column slice (one dependent launch less).
        if (avg_cand && !pair_first && !pair_second && !prep->pair && prep->mc <= 1 && !prep->persist &&
            prep->splits > 1 && uint64_t(prep->splits + 1) * P * Q <= uint64_t(128) * prep->splits) {
          gemm::ConvGeom g{};
          if (implicit) g = gemm::conv_geom(batch, in.h, in.w, cin, k, k, st, pad, P, Q, cg, gi * cg, 0);
          if (implicit ? g.tiles_w == 1 && g.tiles_h == 1 : M <= 128) {
            pout = {reinterpret_cast<uint16_t*>(alloc(uint64_t(batch) * cout * 2)), batch, 1, 1, cout};
            gemm::Epilogue ep = e;
            ep.out = pout.p;
            ep.ldo = uint64_t(cout);
            std::shared_ptr<gemm::Prepared> np;
            if (implicit) {
              g.pool = 3;
              np = std::make_shared<gemm::Prepared>(gemm::prepare_conv(in.p, g, Bop, ep, prep->bn));
            } else {  // a 1x1 conv: one plain M-tile holding all M / HW images
              np = std::make_shared<gemm::Prepared>(
                  gemm::prepare({A, M, uint64_t(kp), uint64_t(cin)}, Bop, ep, prep->bn));
              np->g.pool = 3;
              np->g.P = P;
              np->g.Q = Q;
              np->g.N = batch;
            }
            np->lean = prep->lean;
            np->splits = prep->splits;
            prep = np;
            fused_here = true;
          }
        }
        const uint64_t b_off = w_off + uint64_t(gi) * kg * rsc * 2;
        const bool do_params = first_group && bind_params;
        auto rebind = [=](cudaStream_t s) {
          if (first_group && wpad) pad_rows(wptr(w_off), cout, rsc, wpad, kp, s);
          if (!wpad)
            prep->tb = gemm::make_tmap(wptr(b_off), uint64_t(kg), uint64_t(kp), uint64_t(kp), gemm::b_box_rows(*prep));
          else prep->tb = gemm::make_tmap(wpad + uint64_t(gi) * kg * kp, uint64_t(kg), uint64_t(kp), uint64_t(kp),
                                         gemm::b_box_rows(*prep));
          if (do_params) bind_params(s);
        };
        if (pair_second || gpair_second) {
          auto a = pending->prep;
          auto rb_a = pending->rebind;
          pending.reset();
          if (a->bn == prep->bn && a->lean == prep->lean && (a->bn != 256 || (a->splits == 1 && prep->splits == 1))) {
            // one split count for both; the launch must stay one wave
            int sp = std::min(a->splits, prep->splits);
            const uint64_t t = tile_rows(*a) / 128 * ((a->N + a->bn - 1) / a->bn) +
                               gemm::tile_rows(*prep) / 128 * ((prep->N + prep->bn - 1) / prep->bn);
            while (sp > 1 && t * uint64_t(sp) > uint64_t(sms_)) sp /= 2;
            a->splits = prep->splits = sp;
            auto both = [rb_a, rebind](cudaStream_t s) {
              rb_a(s);
              rebind(s);
            };
            steps_.push_back(std::make_unique<Step>(
                Step{[a, prep](cudaStream_t s) { gemm::run_pair(*a, prep.get(), s); }, both}));
          } else {
            steps_.push_back(std::make_unique<Step>(Step{[a](cudaStream_t s) { gemm::run(*a, s); }, rb_a}));
            steps_.push_back(std::make_unique<Step>(Step{[prep](cudaStream_t s) { gemm::run(*prep, s); }, rebind}));
          }
        } else if (pair_first || gpair_first) {
          pending = Pending{prep, rebind};
        } else {
          steps_.push_back(std::make_unique<Step>(Step{[prep](cudaStream_t s) { gemm::run(*prep, s); }, rebind}));
        }
        if (branch) steps_.back()->branch = nbranches_;
        first_group = false;
      }
      flops_ += 2.0 * double(M) * cout * rsc;
      produced = out;
      if (branch) branch_of[l.s("out")] = nbranches_++;
      if (!l.s("out").empty()) named[l.s("out")] = out;
      if (!branch) cur = out;
      if (fused_here) {  // this conv's tap is the pooled map (the next layer's); its own is not kept
        produced = {};
        cur = pout;
        pool_fused = true;
        if (avg_cand) {  // the pooled [N][C] vector (the next layer, pool_avg, is skipped)
          cur = pout;
        } else if (pool_flat) {  // written NCHW: the flatten step is free
          cur = {pout.p, batch, 1, 1, pout.h * pout.w * pout.c};
          flat_done = true;
        }
      }
    } else if (l.kind == "pool_max") {
      const int k = l.i("k"), st = l.i("stride", k), pad = l.i("pad", 0);
      const Act in = cur;
      const int P = (in.h + 2 * pad - k) / st + 1, Q = (in.w + 2 * pad - k) / st + 1;
      const Act out{reinterpret_cast<uint16_t*>(alloc(uint64_t(batch) * P * Q * in.c * 2)), batch, P, Q, in.c};
      // A pool feeding a flatten writes NCHW itself (the flatten step is then
      // free): one launch less for VGG / AlexNet. TRIMS_POOL_NCHW=0: A/B.
      static const bool pool_nchw_on = [] {
        const char* e = std::getenv("TRIMS_POOL_NCHW");
        return !(e && std::string(e) == "0");
      }();
      const bool nchw = pool_nchw_on && P * Q > 1 && l.s("out").empty() && li + 1 < layers.size() &&
                        layers[li + 1].kind == "flatten";
      steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) {
        nn::maxpool(in.p, out.p, in.n, in.h, in.w, in.c, k, st, pad, P, Q, s, nchw);
      }}));
      if (!l.s("out").empty()) named[l.s("out")] = out;
      if (nchw) {
        cur = {out.p, batch, 1, 1, P * Q * in.c};  // already flattened (NCHW order)
        flat_done = true;
        produced = cur;
      } else {
        cur = out;
      }
    } else if (l.kind == "pool_avg") {
      const Act in = cur;
      const Act out{reinterpret_cast<uint16_t*>(alloc(uint64_t(batch) * in.c * 2)), batch, 1, 1, in.c};
      steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) {
        nn::avgpool_global(in.p, out.p, in.n, in.h * in.w, in.c, s);
      }}));
      cur = out;
    } else if (l.kind == "flatten") {
      const Act in = cur;
      if (flat_done) {  // the pool before already wrote the NCHW-flattened vector
        flat_done = false;
      } else if (in.h * in.w > 1) {  // FC weights expect torch's NCHW flatten order
        const Act out{reinterpret_cast<uint16_t*>(alloc(in.elems() * 2)), batch, 1, 1, in.h * in.w * in.c};
        steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) {
          nn::flatten_nchw(in.p, out.p, in.n, in.h * in.w, in.c, s);
        }}));
        cur = out;
      } else {
        cur = {in.p, batch, 1, 1, in.c};
      }
    } else if (l.kind == "fc") {
      const Act in = cur;
      const int cin = l.i("cin"), cout = l.i("cout");
      if (in.c != cin) raise(Errc::InvalidArgument, l.s("name") + ": fc input mismatch");
      const uint64_t w_off = offset_of(l.s("name") + ".weight");
      float* bias = nullptr;
      uint64_t b_off = 0;
      if (l.i("bias")) {
        bias = reinterpret_cast<float*>(alloc(uint64_t(cout) * 4));
        b_off = offset_of(l.s("name") + ".bias");
      }
      const bool last = int(li) == last_fc;
      const bool relu = l.i("relu") != 0;
      const Act out{reinterpret_cast<uint16_t*>(alloc(uint64_t(batch) * cout * 2)), batch, 1, 1, cout};
      if (last) {
        classes_ = cout;
        logits_ = reinterpret_cast<float*>(alloc(uint64_t(batch) * cout * 4));
      }
      float* lg = last ? logits_ : nullptr;
      const int sms = sms_;
      auto bind_bias = [=](cudaStream_t s) {
        if (bias) bf16_to_f32(wptr(b_off), bias, cout, s);
      };
      if (batch <= 8 && cin % 256 == 0) {  // HBM-bound GEMV: weights streamed once
        steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) {
          nn::gemv(in.p, batch, cin, wptr(w_off), cout, bias, relu, out.p, lg, cout, sms, s);
        }, bind_bias}));
      } else {
        gemm::Epilogue e{out.p, uint64_t(cout), nullptr, bias, nullptr, 0, relu};
        auto prep = std::make_shared<gemm::Prepared>(
            gemm::prepare({in.p, uint64_t(batch), uint64_t(cin), uint64_t(cin)},
                          {reinterpret_cast<const uint16_t*>(uintptr_t(256)), uint64_t(cout), uint64_t(cin),
                           uint64_t(cin)},
                          e));
        prep->lean = lean;
        // batch > 8: few output tiles (one M-tile per 128 images), each
        // streaming a K-long weight slab: split K so the weights stream on
        // most SMs (VGG-16 b32 fc6: 64 CTAs -> 128); latency mode only, as for convs
        if (split_ok)
          prep->splits = gemm::pick_splits(gemm::tile_rows(*prep), uint64_t(cout), uint64_t(cin), prep->bn, sms_);
        auto rebind = [=](cudaStream_t s) {
          prep->tb = gemm::make_tmap(wptr(w_off), uint64_t(cout), uint64_t(cin), uint64_t(cin), gemm::b_box_rows(*prep));
          bind_bias(s);
        };
        steps_.push_back(std::make_unique<Step>(Step{[prep](cudaStream_t s) { gemm::run(*prep, s); }, rebind}));
        if (last) {
          const int n = batch * cout;
          steps_.push_back(std::make_unique<Step>(Step{[=](cudaStream_t s) { nn::bf16_to_f32(out.p, lg, n, s); }}));
        }
      }
      flops_ += 2.0 * double(batch) * cin * cout;
      cur = out;
    } else {
      raise(Errc::InvalidArgument, "unknown layer kind " + l.kind);
    }
    attach_joins();
    if (l.kind != "input") {
      if (l.kind == "fc" && int(li) == last_fc) taps_.push_back({logits_, batch, 1, 1, classes_, 1});
      else if (l.kind == "conv" && !produced.p)
        taps_.push_back({nullptr, 0, 0, 0, 0, 2});  // fused: the following pool's tap holds the result
      else if (l.kind == "conv" || (l.kind == "pool_max" && produced.p))
        taps_.push_back({produced.p, produced.n, produced.h, produced.w, produced.c, 0});
      else taps_.push_back({cur.p, cur.n, cur.h, cur.w, cur.c, 0});
    }
  }
  if (pending) raise(Errc::Internal, "a grouped GEMM was never launched");
  if (!branch_of.empty()) raise(Errc::InvalidArgument, "a branch output is never consumed");
  if (!logits_) raise(Errc::InvalidArgument, "architecture has no fc output");
  for (const auto& s : steps_) launches_ += s->launches;
  for (const auto& f : folds_) max_fold_c_ = std::max(max_fold_c_, f.C);
  if (!folds_.empty()) d_jobs_ = reinterpret_cast<FoldJob*>(alloc(folds_.size() * sizeof(FoldJob)));
  TRIMS_CUDA(cudaStreamCreateWithFlags(&capture_stream_, cudaStreamNonBlocking));
  if (nbranches_) {
    TRIMS_CUDA(cudaStreamCreateWithFlags(&side_stream_, cudaStreamNonBlocking));
    fork_ev_.resize(size_t(nbranches_));
    join_ev_.resize(size_t(nbranches_));
    for (auto* v : {&fork_ev_, &join_ev_})
      for (auto& e : *v) TRIMS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  rebind(weights);
}

Net::~Net() {
  DeviceGuard g(device_, /*nothrow=*/true);
  if (exec_) cudaGraphExecDestroy(exec_);
  if (graph_) cudaGraphDestroy(graph_);
  if (capture_stream_) cudaStreamDestroy(capture_stream_);
  if (side_stream_) cudaStreamDestroy(side_stream_);
  for (auto* v : {&fork_ev_, &join_ev_})
    for (auto e : *v) cudaEventDestroy(e);
  for (void* p : owned_) cudaFree(p);
}

const Net::Tap& Net::tap(int i) const {
  if (i < 0 || i >= int(taps_.size())) raise(Errc::InvalidArgument, "no such layer " + std::to_string(i));
  return taps_[size_t(i)];
}

void Net::rebind(const uint8_t* weights) {
  DeviceGuard g(device_);
  static const bool prof = std::getenv("TRIMS_REBIND_PROFILE") != nullptr;  // diagnostic: phase times to stderr
  const auto t0 = std::chrono::steady_clock::now();
  wbase_ = weights;
  for (const auto& s : steps_)
    if (s->rebind) s->rebind(capture_stream_);
  const auto t1 = std::chrono::steady_clock::now();
  if (!folds_.empty()) {
    std::vector<FoldJob> jobs;
    jobs.reserve(folds_.size());
    auto w = [&](uint64_t off) { return reinterpret_cast<const uint16_t*>(wbase_ + off); };
    for (const auto& f : folds_) jobs.push_back({w(f.og), w(f.ob), w(f.om), w(f.ov), f.scale, f.shift, f.C, 0});
    TRIMS_CUDA(cudaMemcpyAsync(d_jobs_, jobs.data(), jobs.size() * sizeof(FoldJob), cudaMemcpyHostToDevice,
                               capture_stream_));
    nn::bn_fold_batched(d_jobs_, int(jobs.size()), max_fold_c_, 1e-5f, capture_stream_);
  }
  TRIMS_CUDA(cudaStreamSynchronize(capture_stream_));
  const auto t2 = std::chrono::steady_clock::now();
  // Kernel parameters (tensor maps, pointers) changed: re-record the graph
  // and update the instantiated one in place (same topology) instead of
  // instantiating a new executable graph.
  if (exec_) capture_graph();
  if (prof) {
    const auto t3 = std::chrono::steady_clock::now();
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    std::fprintf(stderr, "rebind_us steps=%.1f fold_sync=%.1f graph=%.1f\n", us(t0, t1), us(t1, t2), us(t2, t3));
  }
}

void Net::capture_graph() {
  cudaGraph_t g = nullptr;
  TRIMS_CUDA(cudaStreamBeginCapture(capture_stream_, cudaStreamCaptureModeThreadLocal));
  try {
    record(capture_stream_);
  } catch (...) {  // close the capture so the stream stays usable, report the launch error
    cudaStreamEndCapture(capture_stream_, &g);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    throw;
  }
  TRIMS_CUDA(cudaStreamEndCapture(capture_stream_, &g));
  if (exec_) {
    cudaGraphExecUpdateResultInfo info{};
    if (cudaGraphExecUpdate(exec_, g, &info) == cudaSuccess) {
      if (graph_) cudaGraphDestroy(graph_);
      graph_ = g;
      return;
    }
    cudaGetLastError();  // topology changed: fall back to a fresh instantiation
    cudaGraphExecDestroy(exec_);
    exec_ = nullptr;
  }
  if (graph_) cudaGraphDestroy(graph_);
  graph_ = g;
  TRIMS_CUDA(cudaGraphInstantiate(&exec_, graph_, 0));
}

void Net::record(cudaStream_t stream) {
  for (const auto& s : steps_) {
    for (int j : s->joins) TRIMS_CUDA(cudaStreamWaitEvent(stream, join_ev_[size_t(j)], 0));
    if (s->branch >= 0) {  // fork: the side stream starts from the main stream's current point
      const size_t b = size_t(s->branch);
      TRIMS_CUDA(cudaEventRecord(fork_ev_[b], stream));
      TRIMS_CUDA(cudaStreamWaitEvent(side_stream_, fork_ev_[b], 0));
      s->run(side_stream_);
      TRIMS_CUDA(cudaEventRecord(join_ev_[b], side_stream_));
    } else {
      s->run(stream);
    }
  }
}

void Net::run(cudaStream_t stream, bool use_graph) {
  DeviceGuard g(device_);
  if (!use_graph) {
    record(stream);
    return;
  }
  if (!exec_) capture_graph();
  TRIMS_CUDA(cudaGraphLaunch(exec_, stream));
}

}  // namespace trims::nn
