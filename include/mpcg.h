/*
 * mpcg.h — C ABI of the B200-native 2PC secret-shared inference engine (libmpcg.so).
 *
 * Drop-in boundary for the MPC-Pipe reference's hot path (arXiv 2209.13643). The
 * reference is a header-only C++ library with no FFI; each entry point below replaces
 * the reference interface cited beside it (paths relative to
 * /root/reference/proj/include/mpcpipe). Plain pointers and sizes only; every call
 * returns an mpcg status code, with the message in mpcg_last_error().
 *
 * Status codes mirror the reference exception classes (errors.hpp:8-45):
 *   RangeError=1 ShapeError=2 ConfigError=3 ProtocolError=4 TransportError=5
 *   BudgetError=6 UsageError=7, plus CUDA=8, NCCL=9, internal=10.
 *
 * A session holds the party slots living in this process on one GPU:
 *   n_local = 2: both parties of a 2PC pair on `device` (1-GPU mode)
 *   n_local = 1: party `party` only; connect the peer with mpcg_session_connect_nccl.
 * Tensors carry one u64 share per local slot (slot-major, row-major Z_2^64 words, i.e.
 * the RingTensor layout of ring/tensor.hpp:36-76 repeated per slot).
 * Every op takes the same tag strings as the reference, so the seeded dealer draws the
 * exact triples the reference draws (sharing/triple.hpp:138-151) and per-party output
 * shares are word-identical.
 */
#ifndef MPCG_H
#define MPCG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPCG_OK 0
#define MPCG_ERR_RANGE 1
#define MPCG_ERR_SHAPE 2
#define MPCG_ERR_CONFIG 3
#define MPCG_ERR_PROTOCOL 4
#define MPCG_ERR_TRANSPORT 5
#define MPCG_ERR_BUDGET 6
#define MPCG_ERR_USAGE 7
#define MPCG_ERR_CUDA 8
#define MPCG_ERR_NCCL 9
#define MPCG_ERR_INTERNAL 10

#define MPCG_REDUCE_SUM 0 /* transport/transport.hpp:12 Reduce::Sum */
#define MPCG_REDUCE_XOR 1 /* Reduce::Xor */

typedef struct mpcg_session mpcg_session;
typedef struct mpcg_tensor mpcg_tensor;
typedef struct mpcg_model mpcg_model;
typedef struct mpcg_executor mpcg_executor;
typedef struct mpcg_triple_queue mpcg_triple_queue;

/* Thread-local message of the last failing call. */
const char* mpcg_last_error(void);
int mpcg_version(void);
/* Number of visible CUDA devices (0 on a host without a GPU). */
int mpcg_device_count(int* out);

/* ---- session: replaces SessionConfig + SeededDealer + mask CounterRng + Communicator
 *      (transport/config.hpp:22-39, sharing/triple.hpp:138-151, engine/bench.hpp:39-40,
 *       transport/transport.hpp:51-82). mask_seed keys CounterRng(mask_seed, party). */
int mpcg_session_create(int device, int n_local, int party, uint64_t seed, uint64_t mask_seed, int frac_bits,
                        mpcg_session** out);
int mpcg_session_destroy(mpcg_session* s);
/* ProtoCtx knobs (protocols/context.hpp:17-35): chunks, threshold bytes, merged adder. */
int mpcg_session_set_pipeline(mpcg_session* s, int chunks, uint64_t threshold_bytes, int merged_adder);
/* Emulated link (transport/config.hpp:41-43, sim.hpp:90-92): bandwidth<=0 disables. */
int mpcg_session_set_link(mpcg_session* s, double latency_s, double bandwidth_Bps, double sec_per_message);
/* Data-parallel shard: this pair holds rows [offset, offset+local) of a global batch. */
int mpcg_session_set_shard(mpcg_session* s, uint64_t local_batch, uint64_t global_batch, uint64_t batch_offset);
/* NCCL link for n_local == 1 (the socket mesh of transport/socket.hpp:345-402). */
int mpcg_nccl_unique_id(uint8_t out[128]);
int mpcg_session_connect_nccl(mpcg_session* s, const uint8_t id[128], int rank);
/* TCP link for n_local == 1 (transport/socket.hpp:60-413, SocketComm): party 0 listens on
 * host:port, party 1 connects; both block until paired or `timeout_s` passes. Every payload is a
 * framed message {seq, words, tag hash}; a mismatch raises MPCG_ERR_PROTOCOL at the wait. For
 * parties in different processes or hosts; not capturable into a CUDA graph. */
int mpcg_session_connect_socket(mpcg_session* s, const char* host, int port, double timeout_s);
int mpcg_session_sync(mpcg_session* s);
/* 1-GPU mode: run multi-round chains (ReLU, tournament rounds) as one persistent cooperative
 * kernel (1), one kernel per exchange round (0), or auto by size (2, default). Values are
 * identical in every mode. */
int mpcg_session_set_persistent(mpcg_session* s, int enable);
/* CommStats of one local slot (transport/transport.hpp:39-45): bytes, collectives, p2p. */
int mpcg_session_stats(mpcg_session* s, int slot, uint64_t out[3]);
int mpcg_session_n_local(mpcg_session* s, int* out);
/* Communicator::trace / clear_trace / now / add_delay (transport/transport.hpp:25-82).
 * While enabled, one row per collective: seq, kind, tag, bytes and device timestamps in seconds
 * since the trace was enabled — t[0] issue, t[1] sent (sender occupancy charged), t[2] wait
 * begin, t[3] wait end (occupancy = t1 - t0, stall = t3 - t2; report.hpp:42-66 sums them into
 * delta-wait / linear-comm). Reading synchronises the session. Opens recorded inside a graph
 * capture or performed in-kernel carry no timestamps (0). */
int mpcg_session_trace(mpcg_session* s, int enable);
int mpcg_session_trace_count(mpcg_session* s, uint64_t* n);
int mpcg_session_trace_get(mpcg_session* s, uint64_t i, uint32_t* seq, int* kind, uint64_t* bytes, double t[4],
                           char* tag, int tag_cap);
int mpcg_session_clear_trace(mpcg_session* s);
/* Host wall seconds since the session was created. */
int mpcg_session_now(mpcg_session* s, double* out);
/* Fault injection: the session's compute stream idles `seconds` at this point. */
int mpcg_session_add_delay(mpcg_session* s, double seconds);

/* ---- tensors (device RingTensor shares; ring/tensor.hpp:36-76) ---- */
int mpcg_tensor_create(mpcg_session* s, int ndim, const uint64_t* dims, int scale_bits,
                       const uint64_t* host /* n_local*numel words or NULL */, mpcg_tensor** out);
int mpcg_tensor_download(mpcg_tensor* t, uint64_t* host /* n_local*numel words */);
int mpcg_tensor_shape(const mpcg_tensor* t, int* ndim, uint64_t dims[8], int* scale_bits);
int mpcg_tensor_destroy(mpcg_tensor* t);
/* deal_input_share (engine/executor.hpp:70-75): CounterRng(seed, 0x11a9) over the global
 * input; this session keeps rows [batch_offset, batch_offset + dims[0]). */
int mpcg_deal_input(mpcg_session* s, const double* x_global, int ndim, const uint64_t* global_dims,
                    uint64_t batch_offset, uint64_t local_batch, uint64_t seed, mpcg_tensor** out);

/* ---- protocol ops (protocols/*.hpp, nonlinear/*.hpp). Each returns a new tensor. ---- */
/* Communicator::reveal (transport/transport.hpp:76-79): every slot receives the opening. */
int mpcg_open(mpcg_session* s, const mpcg_tensor* x, int reduce, const char* tag, mpcg_tensor** out);
int mpcg_beaver_mul(mpcg_session* s, const mpcg_tensor* x, const mpcg_tensor* y, const char* tag, int chunks,
                    mpcg_tensor** out);                                        /* beaver.hpp:43 */
int mpcg_beaver_square(mpcg_session* s, const mpcg_tensor* x, const char* tag, int chunks,
                       mpcg_tensor** out);                                     /* beaver.hpp:88 */
int mpcg_beaver_and(mpcg_session* s, const mpcg_tensor* x, const mpcg_tensor* y, const char* tag, int chunks,
                    mpcg_tensor** out);                                        /* beaver.hpp:129 */
int mpcg_beaver_matmul(mpcg_session* s, const mpcg_tensor* x, const mpcg_tensor* y, int transpose_b,
                       const char* tag, int chunks, mpcg_tensor** out);        /* beaver.hpp:186 */
int mpcg_binary_add(mpcg_session* s, const mpcg_tensor* x, const mpcg_tensor* y, int width, int merged,
                    int chunks, const char* tag, mpcg_tensor** out);           /* adder.hpp:237 */
int mpcg_a2b(mpcg_session* s, const mpcg_tensor* x, int chunks, const char* tag, mpcg_tensor** out); /* compare.hpp:24 */
int mpcg_msb(mpcg_session* s, const mpcg_tensor* x, int chunks, const char* tag, mpcg_tensor** out); /* compare.hpp:57 */
int mpcg_b2a_bit(mpcg_session* s, const mpcg_tensor* b, const char* tag, int chunks,
                 mpcg_tensor** out);                                           /* compare.hpp:67 */
int mpcg_less_than(mpcg_session* s, const mpcg_tensor* x, const mpcg_tensor* y, int chunks, const char* tag,
                   mpcg_tensor** out);                                         /* compare.hpp:87 */
int mpcg_truncate(mpcg_session* s, const mpcg_tensor* x, int bits, mpcg_tensor** out); /* trunc.hpp:25 */
int mpcg_relu(mpcg_session* s, const mpcg_tensor* x, const char* tag, mpcg_tensor** out); /* activations.hpp:39 */
int mpcg_max_last_dim(mpcg_session* s, const mpcg_tensor* x, uint64_t L, const char* tag,
                      mpcg_tensor** out);                                      /* activations.hpp:51 */
int mpcg_exp(mpcg_session* s, const mpcg_tensor* x, const char* tag, mpcg_tensor** out); /* approx.hpp:22 */
int mpcg_reciprocal(mpcg_session* s, const mpcg_tensor* x, const char* tag, mpcg_tensor** out); /* approx.hpp:43 */
int mpcg_softmax(mpcg_session* s, const mpcg_tensor* x, uint64_t L, const char* tag,
                 mpcg_tensor** out);                                           /* activations.hpp:93 */
int mpcg_maxpool2d(mpcg_session* s, const mpcg_tensor* x, uint64_t N, uint64_t C, uint64_t H, uint64_t W,
                   uint64_t k, uint64_t stride, const char* tag, mpcg_tensor** out); /* activations.hpp:114 */
/* Extensions (not in the reference, built from its blocks; oracle/mpc_oracle.py restates them). */
int mpcg_sigmoid(mpcg_session* s, const mpcg_tensor* x, const char* tag, mpcg_tensor** out);
int mpcg_gelu(mpcg_session* s, const mpcg_tensor* x, const char* tag, mpcg_tensor** out);
int mpcg_inv_sqrt(mpcg_session* s, const mpcg_tensor* v, const char* tag, int newton_iters, mpcg_tensor** out);
int mpcg_layernorm(mpcg_session* s, const mpcg_tensor* x, uint64_t d, const mpcg_tensor* gamma,
                   const mpcg_tensor* beta, int public_weights, const char* tag, mpcg_tensor** out);
int mpcg_global_avg_pool(mpcg_session* s, const mpcg_tensor* x, uint64_t N, uint64_t C, uint64_t HW,
                         mpcg_tensor** out);

/* ---- TripleSource plugin (sharing/triple.hpp:126-179): offline/online split ----
 * A queue holds materialised 2PC triples, consumed in fetch order with the reference's
 * QueueTripleSource semantics (spec checked -> MPCG_ERR_PROTOCOL "triple queue spec mismatch at
 * record i" / "triple queue exhausted"; tags ignored). Offline: a session in record mode
 * materialises every triple it fetches from its seeded dealer into the queue, or a queue is
 * loaded from a reference triple file (save_triples format, triple.hpp:181-307; records must be
 * valid Beaver triples). Online: a session using the queue reads triples from HBM instead of
 * regenerating them. Queues are device-resident on the session's GPU; not for graph capture or
 * data-parallel shards. */
int mpcg_triple_queue_create(mpcg_triple_queue** out);
int mpcg_triple_queue_destroy(mpcg_triple_queue* q);
int mpcg_triple_queue_size(mpcg_triple_queue* q, uint64_t* records, uint64_t* consumed);
int mpcg_triple_queue_rewind(mpcg_triple_queue* q);
int mpcg_triple_queue_save(mpcg_triple_queue* q, const char* path);   /* save_triples */
int mpcg_triple_queue_load(mpcg_triple_queue* q, const char* path);   /* load_triples (appends) */
int mpcg_session_record_triples(mpcg_session* s, mpcg_triple_queue* q /* NULL stops */);
int mpcg_session_use_triple_queue(mpcg_session* s, mpcg_triple_queue* q /* NULL = seeded dealer */);
/* TripleSource::fetch (triple.hpp:126-130): this session's local party shares of the next triple
 * for the spec (kind 0 arith / 1 binary; matmul; square; transpose_b), from the seeded dealer or
 * the queue in use. Returns three tensors (a, b, c), one share per local slot. */
int mpcg_dealer_fetch(mpcg_session* s, int kind, int matmul, int square, int transpose_b, int nda,
                      const uint64_t* dims_a, int ndb, const uint64_t* dims_b, const char* tag, mpcg_tensor** a,
                      mpcg_tensor** b, mpcg_tensor** c);

/* ---- model + executor (engine/model.hpp, engine/executor.hpp:173-205) ---- */
#define MPCG_LAYER_DENSE 0
#define MPCG_LAYER_CONV2D 1
#define MPCG_LAYER_RELU 2
#define MPCG_LAYER_MAXPOOL2D 3
#define MPCG_LAYER_FLATTEN 4
#define MPCG_LAYER_ATTENTION 5
#define MPCG_LAYER_SOFTMAX 6
#define MPCG_LAYER_MEANPOOL 7
/* Extensions (not in the reference; needed by the ResNet-18 / BERT-base configs). */
#define MPCG_LAYER_ADD 8
#define MPCG_LAYER_GLOBAL_AVG_POOL 9
#define MPCG_LAYER_GELU 10
#define MPCG_LAYER_LAYERNORM 11
int mpcg_model_create(const char* name, int frac_bits, int ndim, const uint64_t* input_dims, mpcg_model** out);
int mpcg_model_add_layer(mpcg_model* m, const char* name, int kind, uint64_t out, uint64_t kernel,
                         uint64_t stride, uint64_t pad, uint64_t heads, int bias);
/* Extension: add_layer with wiring — `from` = the layer whose output it reads (NULL/"" = the
 * previous layer, "input" = the model input), `with_` = an ADD's second operand. (The
 * reference's models are chains, engine/model.hpp:18-20; add_layer == add_layer_ex(.., 0, 0).) */
int mpcg_model_add_layer_ex(mpcg_model* m, const char* name, int kind, uint64_t out, uint64_t kernel,
                            uint64_t stride, uint64_t pad, uint64_t heads, int bias, const char* from,
                            const char* with_);
int mpcg_model_destroy(mpcg_model* m);
/* ExecOptions (engine/executor.hpp:28-36). */
int mpcg_executor_create(mpcg_session* s, const mpcg_model* m, int public_weights, int pipelined, int chunks,
                         uint64_t chunk_threshold, int merged_adder, mpcg_executor** out);
/* deal_weight_shares / public_weight_set (engine/executor.hpp:49-68). */
int mpcg_executor_deal_weights(mpcg_executor* e, int count, const char* const* names,
                               const double* const* values, const uint64_t* counts /* doubles per tensor */,
                               uint64_t seed);
/* Extension (north_star (3)): in pipelined mode also open the linear layers' activation side in
 * `chunks` row blocks ("<tag>.eps.chunk<k>", the beaver_matmul chunk unit of
 * protocols/beaver.hpp:197-250) for operands >= the chunk threshold, each block's combine GEMM
 * running as it lands. Off (default) = the reference's unchunked weight_matmul (executor.hpp:305);
 * values and bytes are identical either way, only the collective count differs. */
int mpcg_executor_set_linear_chunks(mpcg_executor* e, int on);
int mpcg_executor_run(mpcg_executor* e, const mpcg_tensor* input, mpcg_tensor** out); /* executor.hpp:193 */
/* CUDA-graph form of run(): capture one steady-state inference that reads `input` in place
 * (pipelined mode needs one mpcg_executor_run first), then each replay performs the next
 * inference with fresh dealer triples (same values as successive run() calls). The
 * replay output is valid until the next replay. */
int mpcg_executor_capture(mpcg_executor* e, const mpcg_tensor* input);
int mpcg_executor_replay(mpcg_executor* e, mpcg_tensor** out);
/* While a graph is held, eager runs and the session's other triple-fetching ops fail with
 * MPCG_ERR_USAGE (the graph owns the dealer streams). Releasing it hands them back: the next
 * run() continues the iteration sequence where the last replay left it. */
int mpcg_executor_release_graph(mpcg_executor* e);
/* Per-layer device times (ms) of the next runs: enable=1 turns timing on. */
int mpcg_executor_time_layers(mpcg_executor* e, int enable);
int mpcg_executor_layer_times(mpcg_executor* e, int max, float* ms, int* count);
int mpcg_executor_destroy(mpcg_executor* e);

/* Ring-GEMM engine: 0 = SIMT only, 1 = tcgen05 int8-limb path for every shape within its
 * exact-accumulation budget (K' <= 16384), 2 = auto (tcgen05 for large shapes; default),
 * 3 = as 1 but one CTA per party slot only (the both-slots combine kernel off). */
int mpcg_set_gemm_mode(int mode);
/* 1-GPU mode: pair evaluation (1, default: one thread evaluates both local party slots of an
 * element and writes each open's opened value once; summed eps/delta opens) or per-slot
 * kernels (0: each slot writes its own payload and reads the peer's, as two separate parties
 * do). Values are identical. Process-wide; affects kernels launched or captured afterwards. */
int mpcg_set_pair_eval(int on);
/* Small-M combines (M <= 16, unbatched): fused-segment streaming kernel (1, default) or the
 * tiled SIMT/tcgen05 paths (0). */
int mpcg_set_gemv(int on);
/* Debug: stage timestamps (clock64) of the last tcgen05 GEMM's first CTA when MPCG_TC2_TRACE=1;
 * [stage][10] = MMA wait start/end/issue end, generated-producer and memory-producer
 * empty-wait start/end/arrive. */
int mpcg_debug_tc2_trace(uint64_t* out, int n);
/* Debug: per-stage clock64 stamps of CTA (0,0,0) of the last both-slots tcgen05 GEMM run with
 * MPCG_TC3_TRACE=1 ([256][8]: MMA wait/full/issued, producer start/wait/acquired/arrived). */
int mpcg_debug_tc3_trace(uint64_t* out, int n);
/* Measurement: the dealer's draw rate on `device` — splitmix64 counter draws (rng.hpp) per
 * second, a full grid of independent streams, best of 3 (the ALU roofline of the
 * element-by-element compare chain). */
int mpcg_debug_draw_peak(int device, double* draws_per_s);
/* Link two single-party sessions (party 0, party 1) of this process on the same GPU: the
 * one-party-per-GPU code path with device copies in place of NCCL send/recv. Each party
 * must be driven by its own host thread (a collective waits for the peer's matching post). */
int mpcg_session_connect_loopback(mpcg_session* a, mpcg_session* b);
/* Device-initiated link between party 0's and party 1's single-party sessions of this process
 * (same GPU, or two GPUs with peer access over NVLink): each open's payload is stored by the
 * sender straight into the receiver's inbox and published with a system-scope release flag the
 * receiver's stream acquires on the device — no host event crosses the parties. Capturable into
 * CUDA graphs (flag values follow the replay counter; each replay ends with a device barrier).
 * Each party must be driven by its own host thread. */
int mpcg_session_connect_p2p(mpcg_session* a, mpcg_session* b);

/* ---- measurement hooks (bench.py) ---- */
/* Kernels launched by this library since load. */
uint64_t mpcg_launch_count(void);
/* Time every launch of one kernel class with CUDA events (1 = SPK adder level rounds,
 * 2 = ring GEMM); stop returns total device ms, launches and algorithmic units
 * (bytes for elementwise classes, ring MACs for GEMM). */
int mpcg_probe_start(int kernel_class);
int mpcg_probe_stop(double* total_ms, uint64_t* launches, double* units);
/* Page-locked host buffers and async H2D copies into an existing tensor (e2e path). */
int mpcg_pinned_alloc(uint64_t bytes, void** out);
int mpcg_pinned_free(void* p);
int mpcg_tensor_copy_from_host(mpcg_tensor* t, const uint64_t* host /* n_local*numel words */);
/* Evict L2 between timed steps: memset of a 256 MiB scratch buffer on the session stream. */
int mpcg_session_flush_l2(mpcg_session* s);
/* Device timer on the session stream: start/stop pairs accumulate; ms returns the sum. */
int mpcg_session_timer(mpcg_session* s, int op /* 0 start, 1 stop, 2 reset, 3 read */, double* total_ms);

/* FNV-1a over little-endian words (engine/report.hpp:18-23). */
uint64_t mpcg_fnv1a_words(const uint64_t* words, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif /* MPCG_H */
