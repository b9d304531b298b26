// Model graph + secure executor (H/engine/model.hpp, H/engine/executor.hpp).
#pragma once

#include <optional>

#include "core.hpp"

namespace mpcg {

// Dense..MeanPool are the reference's kinds (H/engine/model.hpp:21); Add..LayerNorm are the
// extensions the ResNet-18 / BERT-base configs need (not in the reference, see ext.cu).
enum class LayerKind : int {
  Dense = 0, Conv2d, Relu, Maxpool2d, Flatten, Attention, Softmax, MeanPool,
  Add, GlobalAvgPool, Gelu, LayerNorm
};

struct LayerSpec {
  std::string name;
  LayerKind kind = LayerKind::Dense;
  size_t out = 0, kernel = 0, stride = 1, pad = 0, heads = 0;
  bool bias = true;
  std::string from;  // extension: input = this earlier layer's output ("input" = model input)
  std::string with;  // extension: second operand of Add
};

struct ModelGraph {
  std::string name = "model";
  int frac_bits = 20;
  Shape input;  // leading dim is the batch
  std::vector<LayerSpec> layers;
};

// Producer index of each layer's input (-1 = model input) and of an Add's second operand.
struct LayerWiring {
  std::vector<long> src, other;
};
LayerWiring layer_wiring(const ModelGraph& g);


std::vector<Shape> infer_shapes(const ModelGraph& g);
std::vector<std::pair<std::string, Shape>> model_weight_shapes(const ModelGraph& g);

// Host-side CounterRng (H/sharing/rng.hpp:10-32), used only at setup (dealing).
struct HostRng {
  u64 key, ctr = 0;
  HostRng(u64 k, u64 stream = 0) : key(k ^ (stream * kPhi)) {}
  u64 operator()() { return drw(key, ++ctr); }
};

struct ExecOptions {
  bool pipelined = false;
  int chunks = 4;
  u64 chunk_threshold = u64(2) << 20;
  bool merged_adder = true;
  // Extension: also chunk the linear layers' activation-side opening (inner-layer pipeline on
  // conv / dense, `north_star` (3)). Off = the reference's unchunked weight_matmul traffic.
  bool linear_chunks = false;
};

struct LayerTiming {  // per-layer device time of the last timed run (ms)
  std::string name;
  float ms = 0;
};

class SecureExecutor {
 public:
  SecureExecutor(Session& s, ModelGraph g, bool public_weights, ExecOptions opt);
  ~SecureExecutor();

  // Weights: every party derives its share from the session seed, standing in for the
  // weight owner's dealer (H/engine/executor.hpp:49-68). `values` in sorted-name order.
  // `counts[i]` = number of doubles behind values[i]; checked against the model's shapes
  // (check_weights, H/engine/model.hpp:366-376) before anything is read.
  void deal_weights(const std::vector<std::string>& names, const std::vector<const double*>& values,
                    const std::vector<size_t>& counts, u64 seed);
  void set_weight(const std::string& name, const u64* host_words);  // n_local*numel (or numel public)

  DT run(const DT& input);

  // CUDA-graph capture of one steady-state inference reading `input` in place (refill it
  // with mpcg_tensor_copy_from_host between replays). replay() returns the arena-backed
  // logits, valid until the next replay. Values equal the eager run's, iteration by
  // iteration (device key table refreshed per replay).
  void capture(const DT& input);
  DT replay();
  // Destroy the captured graph; run() and the session's other ops may fetch triples again
  // (while a graph is held they throw UsageError: the graph owns the dealer streams).
  void release_graph();
  DT graph_out_;
  bool captured_ = false;

  std::vector<std::string> linear_tags() const;
  std::vector<LayerTiming> timings;
  bool time_layers = false;   // per-layer CUDA events (also captured into the graph)
  void collect_timings();

  const ModelGraph& graph() const { return g_; }
  const std::vector<Shape>& shapes() const { return shapes_; }

 public:  // internal (extended __device__ lambdas need public enclosing members)
  struct WeightOp {
    std::string tag, wkey, bkey;
    Shape x_shape;
    TripleSpec spec;
    std::optional<Triple> triple;
    std::optional<Open> delta;
    std::shared_ptr<Block> dbuf_out, dbuf_in;  // persistent delta payload (fixed address across runs)
  };
  void add_weight_op(const std::string& tag, const std::string& wkey, const std::string& bkey, Shape x_shape);
  void build_weight_ops();
  void prepare(size_t i);
  // x source: plain 2-D shares, or an NCHW tensor gathered by im2col when geom != null
  DT weight_matmul(size_t i, const DT& x, const struct ConvGeom* geom, bool col2im_out, Shape out_shape,
                   const DT* addend = nullptr);
  DT attention(const LayerSpec& l, const DT& x, const Shape& in_shape, const DT* addend = nullptr);
  DT run_layer(const LayerSpec& l, const DT& x, const Shape& in_shape, const DT* addend = nullptr);
  DT scale_and_rescale(const DT& x, double c);

  Session& s_;
  ModelGraph g_;
  std::vector<Shape> shapes_;
  bool public_;
  ExecOptions opt_;
  std::map<std::string, DT> w_;
  std::vector<WeightOp> wops_;
  std::map<std::string, size_t> wop_index_;
  std::vector<cudaEvent_t> ev_;
};

}  // namespace mpcg
