// nn.hpp — forward-pass kernels (K8) and the network executor that runs a
// CNN on weights lent by the store (K7 GEMMs + K8 layers, CUDA-graph replay).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "format.hpp"
#include "gemm.hpp"

namespace trims::nn {

void input_prep(const float* in_nchw, uint16_t* out_nhwc, int N, int C, int H, int W, cudaStream_t s);
// groups > 1: that many consecutive channel groups (from c_off) in one launch,
// group g's columns at A + g * N*P*Q * Kp
void im2col(const uint16_t* in, uint16_t* A, int N, int H, int W, int Ctot, int c_off, int Cg, int R, int S, int stride,
            int pad, int P, int Q, int Kp, cudaStream_t s, int groups = 1);
// nchw: write NCHW (the flatten order of a following FC) instead of NHWC.
void maxpool(const uint16_t* in, uint16_t* out, int N, int H, int W, int C, int k, int stride, int pad, int P, int Q,
             cudaStream_t s, bool nchw = false);
void avgpool_global(const uint16_t* in, uint16_t* out, int N, int HW, int C, cudaStream_t s);
// im2col straight from the fp32 NCHW network input (the first conv): fuses the
// input layout/precision prep into the column build. Columns in (r, s, c)
// order, zero beyond R*S*C up to Kp (Kp % 8 == 0).
void im2col_input(const float* in_nchw, uint16_t* A, int N, int C, int H, int W, int R, int S, int stride, int pad,
                  int P, int Q, int Kp, cudaStream_t s);
void flatten_nchw(const uint16_t* in, uint16_t* out, int N, int HW, int C, cudaStream_t s);
void gemv(const uint16_t* x, int M, int K, const uint16_t* W, int N, const float* bias, bool relu, uint16_t* out_bf,
          float* out_f32, int ldo, int sms, cudaStream_t s);
// Batched BN fold at bind time: every BN layer of a network in one launch.
struct FoldJob {
  const uint16_t *gamma, *beta, *mean, *var;
  float *scale, *shift;
  int C, pad_;
};
void bn_fold_batched(const FoldJob* d_jobs, int njobs, int max_c, float eps, cudaStream_t s);
void bn_fold(const uint16_t* gamma, const uint16_t* beta, const uint16_t* mean, const uint16_t* var, float eps, int C,
             float* scale, float* shift, cudaStream_t s);
void bf16_to_f32(const uint16_t* in, float* out, int n, cudaStream_t s);
void pad_rows(const uint16_t* in, int rows, int k, uint16_t* out, int kp, cudaStream_t s);
void softmax(const float* in, float* out, int M, int N, cudaStream_t s);

// One bound network: an architecture (text, one layer per line, written by
// paper_1811_09732_b200/models.py) over a resident manifest whose bf16 KRSC
// weights live at `weights` (the store's segment, mapped read-only), plus a
// private workspace: activations, im2col scratch, folded BN parameters.
// Executor modes (trims_net_create_ex flags).
constexpr int kNetThroughput = 1;  // no split-K: one CTA per output tile (many clients on one GPU)
constexpr int kNetLean = 2;        // throughput + GEMM variants that fit 2 CTAs per SM

class Net {
 public:
  Net(int device, const std::string& arch, const fmt::Manifest& resident, const uint8_t* weights, int batch,
      int flags = 0);
  ~Net();
  float* input() const { return input_; }    // fp32 NCHW [batch, 3, H, W]
  float* logits() const { return logits_; }  // fp32 [batch, classes]
  int classes() const { return classes_; }
  int input_hw() const { return in_hw_; }
  uint64_t input_bytes() const { return uint64_t(batch_) * in_c_ * in_hw_ * in_hw_ * sizeof(float); }
  uint64_t logits_bytes() const { return uint64_t(batch_) * classes_ * sizeof(float); }
  int device() const { return device_; }
  // One forward pass on `stream`; with use_graph the launch sequence is
  // captured once into a CUDA graph and replayed.
  void run(cudaStream_t stream, bool use_graph);
  // Point the executor at another generation of the same resident model
  // (identical manifest, new segment): recomputes weight-dependent state only.
  void rebind(const uint8_t* weights);
  // Output buffer of architecture layer `i` (0-based, the input line excluded)
  // as written by the last forward: NHWC [n, h, w, c]; dtype 0 = bf16, 1 = fp32
  // (the logits). Every layer owns its output buffer, so all taps of one
  // forward stay readable until the next one. For parity tests.
  struct Tap {
    const void* p{nullptr};
    int n{0}, h{0}, w{0}, c{0}, dtype{0};
  };
  const Tap& tap(int i) const;
  int layers() const { return int(taps_.size()); }
  double flops() const { return flops_; }
  uint32_t launches() const { return launches_; }
  uint64_t workspace_bytes() const { return ws_bytes_; }

 private:
  struct Step;
  void record(cudaStream_t stream);
  uint8_t* alloc(uint64_t bytes);

  int device_, batch_, sms_{148};
  const uint8_t* wbase_{nullptr};  // current weights generation (resident blob base)
  int in_hw_{224}, in_c_{3}, classes_{1000};
  std::vector<std::unique_ptr<Step>> steps_;
  std::vector<Tap> taps_;
  std::vector<void*> owned_;
  float* input_{nullptr};
  float* logits_{nullptr};
  double flops_{0};
  uint32_t launches_{0};
  uint64_t ws_bytes_{0};
  cudaGraph_t graph_{nullptr};
  cudaGraphExec_t exec_{nullptr};
  cudaStream_t capture_stream_{nullptr};
  // independent branches (ResNet shortcuts) run on a side stream, fork/join by events
  int nbranches_{0};
  cudaStream_t side_stream_{nullptr};
  std::vector<cudaEvent_t> fork_ev_, join_ev_;
  // BN folds of every layer, batched into one launch per rebind: offsets of
  // gamma/beta/mean/var in the resident blob + destination buffers.
  struct Fold {
    uint64_t og, ob, om, ov;
    float *scale, *shift;
    int C;
  };
  std::vector<Fold> folds_;
  FoldJob* d_jobs_{nullptr};
  int max_fold_c_{0};
  void capture_graph();
};

}  // namespace trims::nn
