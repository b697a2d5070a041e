/* moses_gpu.h — C ABI of the B200-native Moses cost-model hot path.
 *
 * This is the drop-in boundary under the reference's C++ API (namespace
 * moseslab, /root/reference/proj/include/moseslab/{model,lottery,search}.hpp).
 * Every entry point cites the reference function it replaces. Plain pointers
 * and sizes only; no torch or Eigen types. Host buffers are float64 like the
 * reference's Eigen::MatrixXd / VectorXd; "_device" variants take device
 * pointers for bulk work.
 *
 * Layout conventions (identical to the reference):
 *   - flat parameter order (lottery.hpp:13-14): per level, the weight array in
 *     Eigen column-major storage order (element (o,i) of the out x in matrix
 *     at off + i*out + o), then the bias; momentum in the same order.
 *   - feature matrices are row-major n x D (the reference's Eigen matrices are
 *     column-major; the C++ wrapper transposes).
 *
 * Status: 0 = MOSES_OK; 1..25 = 1 + moseslab::ErrorCode ordinal
 * (errors.hpp:10-36) with the same validation order as the reference;
 * >= 100 = library errors. moses_last_error() gives the thread's message.
 *
 * Threading: every handle owns one CUDA stream and its workspaces; handles
 * are independent, so callers may use distinct handles from distinct host
 * threads (the reference's compare pool, tuner.cpp:331-374). A single handle
 * must not be used concurrently (update ops need exclusive access, SPEC.md).
 */
#ifndef MOSES_GPU_H_
#define MOSES_GPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOSES_API __attribute__((visibility("default")))

enum {
  MOSES_OK = 0,
  MOSES_ERR_INVALID_TASK = 1,          /* ErrorCode::InvalidTask */
  MOSES_ERR_INVALID_CONFIG = 2,        /* ErrorCode::InvalidConfig */
  MOSES_ERR_SPACE_TOO_LARGE = 3,       /* ErrorCode::SpaceTooLarge */
  MOSES_ERR_IMMUTABLE_SPACE = 4,       /* ErrorCode::ImmutableSpace */
  MOSES_ERR_BAD_DIMS = 5,              /* ErrorCode::BadDims */
  MOSES_ERR_DIM_MISMATCH = 6,          /* ErrorCode::DimMismatch */
  MOSES_ERR_SHAPE_MISMATCH = 7,        /* ErrorCode::ShapeMismatch */
  MOSES_ERR_VERSION_MISMATCH = 8,      /* ErrorCode::VersionMismatch */
  MOSES_ERR_CORRUPT_STREAM = 9,        /* ErrorCode::CorruptStream */
  MOSES_ERR_EMPTY_DATASET = 10,        /* ErrorCode::EmptyDataset */
  MOSES_ERR_INVALID_RATIO = 11,        /* ErrorCode::InvalidRatio */
  MOSES_ERR_UNNORMALIZED_THRESHOLD = 12, /* ErrorCode::UnnormalizedThreshold */
  MOSES_ERR_ADVERSARY_DISABLED = 13,   /* ErrorCode::AdversaryDisabled */
  MOSES_ERR_UNSTABLE_DECAY = 14,       /* ErrorCode::UnstableDecay */
  MOSES_ERR_INFEASIBLE_SPLIT = 15,     /* ErrorCode::InfeasibleSplit */
  MOSES_ERR_ZERO_MEAN = 16,            /* ErrorCode::ZeroMean */
  MOSES_ERR_INSUFFICIENT_BATCHES = 17, /* ErrorCode::InsufficientBatches */
  MOSES_ERR_PARSE = 22,                /* ErrorCode::ParseError */
  MOSES_ERR_MISSING_FIELD = 23,        /* ErrorCode::MissingField */
  MOSES_ERR_IO = 24,                   /* ErrorCode::IoError */
  MOSES_ERR_CUDA = 100,
  MOSES_ERR_NO_DEVICE = 101,
  MOSES_ERR_CAPACITY = 102,
  MOSES_ERR_INVALID_ARG = 103
};

/* GEMM operand precision.
 *   BF16   single bf16 operands (throughput mode; ~5e-3 from the fp64 reference on the cost model).
 *   TF32   kind::tf32 operands (~5e-4 on predictions, ~2e-3 on gradients).
 *   FP32   3xTF32 split operands (hi*hi + hi*lo + lo*hi on kind::tf32): fp32-level accuracy (the <= 1e-5
 *          parity path); host-API inputs (and device fp32 rows), no training graphs.
 *   BF16X3 split bf16 operands: every operand is hi + lo with hi = rn_bf16(v), lo = rn_bf16(v - hi),
 *          products A_hi*B_hi + A_hi*B_lo + A_lo*B_hi on the bf16 tensor cores (~1e-5 from the fp64
 *          reference: inside the north-star 1e-3 tensor-core bound). Fused 512-wide chain kernels only:
 *          hidden widths 512, input width <= 512. Device-resident input rows are fp32.
 * Device-resident input rows (moses_*_device, training graphs, plans) are bf16 for BF16 handles and
 * fp32 otherwise, with the row stride moses_packed_ld. */
enum { MOSES_PREC_BF16 = 0, MOSES_PREC_TF32 = 1, MOSES_PREC_FP32 = 2, MOSES_PREC_BF16X3 = 3 };
enum { MOSES_MODE_THRESHOLD = 1, MOSES_MODE_RATIO = 2 };        /* PartitionMode, "MOSK" mode byte */
enum { MOSES_DTYPE_F32 = 0, MOSES_DTYPE_BF16 = 1, MOSES_DTYPE_F64 = 2 };

typedef struct moses_model* moses_model_t;
typedef struct moses_adversary* moses_adversary_t;
typedef struct moses_records* moses_records_t;

MOSES_API const char* moses_last_error(void);
MOSES_API const char* moses_version(void);
/* Number of kernels this library launched in the calling process (evidence counter). */
MOSES_API int64_t moses_kernel_launches(void);
MOSES_API int moses_device_check(void);

/* ------------------------------------------------------------------ model (model.hpp:19-25, 51-100) */
/* param_count (model.cpp:141-145). Returns -status on bad dims. */
MOSES_API int64_t moses_param_count(const int32_t* dims, int32_t ndims);
/* init_random (model.cpp:147-167): Glorot-uniform from keyed SplitMix64, bit-exact with the reference.
 * strict = 1 enforces the reference's 4-level rule; 0 allows {D, h1..hL, 1}. Host-side. */
MOSES_API int moses_init_random(const int32_t* dims, int32_t ndims, uint64_t seed, int32_t strict, double* flat_out);
/* Device handle for a model of the given dims. max_rows bounds rows per call (batch + replay). */
MOSES_API int moses_model_create(const int32_t* dims, int32_t ndims, int32_t precision, int64_t max_rows,
                                 moses_model_t* out);
MOSES_API int moses_model_destroy(moses_model_t m);
MOSES_API int moses_model_upload(moses_model_t m, const double* params, const double* momentum, int64_t count);
MOSES_API int moses_model_download(moses_model_t m, double* params, double* momentum, int64_t count);
/* Value-semantics copy (tuner.cpp:349 copies the model per job). dst must have identical dims. */
MOSES_API int moses_model_copy(moses_model_t dst, moses_model_t src);
MOSES_API int moses_model_synchronize(moses_model_t m);

/* predict (model.cpp:169-175): scores for n x D row-major features. */
MOSES_API int moses_predict(moses_model_t m, const double* features, int64_t n, int32_t D, double* scores);
/* penultimate_activations (model.cpp:177-183): n x dims[L-1] row-major out. */
MOSES_API int moses_penultimate(moses_model_t m, const double* features, int64_t n, int32_t D, double* hidden);
/* Bulk scoring on device buffers (candidate pool, cfg4): x_dev is n rows of `ldx` elements of `dtype`
 * already in the packed layout (column D == 1, columns > D zero; see moses_packed_ld). Any n (chunked). */
MOSES_API int moses_predict_device(moses_model_t m, const void* x_dev, int32_t dtype, int64_t ldx, int64_t n,
                                   float* scores_dev);
/* Row stride (elements) of the packed layout for input width D under the handle's precision. */
MOSES_API int64_t moses_packed_ld(moses_model_t m);
/* Per-program scores with segment-sum pooling over statement rows (north-star extension; with all
 * segment lengths 1 this is predict). offsets: programs+1 CSR offsets into the n statement rows. */
MOSES_API int moses_predict_pooled(moses_model_t m, const double* stmt_features, int64_t n, int32_t D,
                                   const int64_t* offsets, int64_t programs, double* scores);

/* gradients (model.cpp:192-244). Result stays on the device (read with moses_gradients_download).
 * adv may be NULL; beta == 0 or NULL adversary skips the confusion term bit-exactly. */
MOSES_API int moses_gradients(moses_model_t m, const double* features, const double* labels, int64_t n, int32_t D,
                              moses_adversary_t adv, double beta, double* loss_out);
/* gradients() on device-resident packed rows (x_dev, ldx) and fp32 labels; no adversary. */
MOSES_API int moses_gradients_device(moses_model_t m, const void* x_dev, int64_t ldx, const float* y_dev, int64_t n,
                                     double* loss_out);
/* gradients with segment-sum pooling (north-star (2)): n_stmt statement rows, `programs` programs with CSR
 * offsets, one label per program. With all segments of length 1 this is moses_gradients. */
MOSES_API int moses_gradients_pooled(moses_model_t m, const double* stmt_features, int64_t n_stmt, int32_t D,
                                     const int64_t* offsets, int64_t programs, const double* labels, double* loss_out);
/* tuner.cpp:146-147 (gradients + momentum apply_update) over host float64 statement rows, queued
 * asynchronously (pipelined: the upload of the next batch overlaps this step's kernels). Returns once
 * queued; x / offsets / y must stay valid and unchanged until the step completes. loss_out (host
 * memory or NULL) receives the step's loss from a per-slot mailbox the step's last kernel writes: by
 * the third following call on the handle at the latest (three staging slots), or by moses_model_synchronize, which waits
 * for every queued step. bf16 handles; capacity max_rows statement rows per step. */
MOSES_API int moses_train_step_pooled_async(moses_model_t m, const double* stmt_features, int64_t n_stmt, int32_t D,
                                            const int64_t* offsets, int64_t programs, const double* labels,
                                            double learning_rate, double momentum, double* loss_out);
MOSES_API int moses_gradients_download(moses_model_t m, double* grads, int64_t count);
MOSES_API int moses_gradients_upload(moses_model_t m, const double* grads, int64_t count);
/* objective (model.cpp:246-261) */
MOSES_API int moses_objective(moses_model_t m, const double* features, const double* labels, int64_t n, int32_t D,
                              moses_adversary_t adv, double beta, double* out);
/* apply_update (model.cpp:263-296) with the device gradients. mask: NULL or count host bytes. */
MOSES_API int moses_apply_update(moses_model_t m, double learning_rate, double momentum, const uint8_t* mask,
                                 int64_t mask_len, int32_t use_momentum);
/* One offline pretraining step (tuner.cpp:146-147): gradients + momentum update. */
MOSES_API int moses_train_step(moses_model_t m, const double* features, const double* labels, int64_t n, int32_t D,
                               double learning_rate, double momentum, double* loss_out);
/* Same on device-resident rows (packed layout, labels fp32); loss stays on device unless loss_out != NULL. */
MOSES_API int moses_train_step_device(moses_model_t m, const void* x_dev, int64_t ldx, const float* y_dev, int64_t n,
                                      double learning_rate, double momentum, double* loss_out);
/* CUDA graph of one device-resident training step over a packed dataset of n_batches x batch rows
 * (row stride = moses_packed_ld): gather batch (device-side index) -> gradients [-> momentum update].
 * with_update = 0 leaves the update to the caller (data parallel: all-reduce the gradients first).
 * Each launch replays `steps` steps; the batch index advances on the device. */
MOSES_API int moses_train_graph_create(moses_model_t m, const void* x_base, int64_t ldx, const float* y_base,
                                       int64_t n_batches, int64_t batch, double learning_rate, double momentum,
                                       int32_t with_update);
/* TenSet-shaped variant: programs of variable statement counts. prog_off_dev: device int64 CSR offsets of
 * every program's statement rows in x_base (n_batches * batch_programs + 1 entries); rows_pad >= the largest
 * batch's statement count (GEMM row count captured in the graph; padding rows carry no gradient).
 * Two graphs alternate between two batch buffers: each step computes on one while a side branch
 * gathers the next batch into the other (batch 0 is gathered here). */
MOSES_API int moses_train_graph_create_pooled(moses_model_t m, const void* x_base, int64_t ldx, const float* y_base,
                                              const int64_t* prog_off_dev, int64_t n_batches, int64_t batch_programs,
                                              int64_t rows_pad, double learning_rate, double momentum,
                                              int32_t with_update);
MOSES_API int moses_train_graph_launch(moses_model_t m, int64_t steps);
MOSES_API int moses_train_graph_kernels(void);
/* ranking_accuracy (model.cpp:298-312): nb batches, rows [off[b], off[b+1]) of features/labels. */
MOSES_API int moses_ranking_accuracy(moses_model_t m, const double* features, const double* labels,
                                     const int64_t* batch_offsets, int32_t nbatches, int32_t D, double* accuracy,
                                     int64_t* pairs, int64_t* concordant);
/* pairwise_ranking_loss (model.cpp:185-190), standalone on host buffers. */
MOSES_API int moses_ranking_loss(const double* scores, const double* labels, int64_t n, double* loss,
                                 int64_t* pairs);
/* Masked Adam on the device gradients (north-star extension; parity pinned by the oracle only). */
MOSES_API int moses_adam_update(moses_model_t m, double lr, double beta1, double beta2, double eps, int32_t step,
                                const uint8_t* mask, int64_t mask_len);

/* ------------------------------------------------------------------ lottery (lottery.hpp:44-83) */
/* xi_scores (lottery.cpp:35-57) from the handle's params and device gradients; xi_out may be NULL. */
MOSES_API int moses_xi_scores(moses_model_t m, int32_t normalize, double* xi_out, int64_t count);
/* partition (lottery.cpp:59-90) over the xi computed by the last moses_xi_scores (or uploaded with
 * moses_xi_upload). The mask is kept on the device; mask_out (count bytes) may be NULL. */
MOSES_API int moses_partition(moses_model_t m, int32_t mode, double value, int32_t phase, uint8_t* mask_out,
                              int64_t count, int64_t* popcount);
MOSES_API int moses_xi_upload(moses_model_t m, const double* xi, int64_t count, int32_t normalized);
MOSES_API int moses_mask_upload(moses_model_t m, const uint8_t* mask, int64_t count);
/* transferable_step (lottery.cpp:92-97) with the device mask and gradients. */
MOSES_API int moses_transferable_step(moses_model_t m, double alpha);
/* variant_decay (lottery.cpp:99-120) with the device mask. */
MOSES_API int moses_variant_decay(moses_model_t m, double alpha, double lambda);
/* The Moses adaptation step fused (tuner.cpp:258-262): xi -> partition -> step -> decay in one
 * device pass sequence; threshold mode normalises xi like the tuner does. */
MOSES_API int moses_lottery_step(moses_model_t m, int32_t mode, double value, int32_t phase, double alpha,
                                 double lambda, uint8_t* mask_out, int64_t count, int64_t* popcount);
/* The same fused step with masked Adam on the transferable scalars (the north star's Adam variant;
 * adam_update arithmetic of moses_adam_update, bias corrections of `step`); variant scalars decay by
 * 1 - lr * lambda. Moments live on the handle (zero at first use). */
MOSES_API int moses_lottery_step_adam(moses_model_t m, int32_t mode, double value, int32_t phase, double lr,
                                      double beta1, double beta2, double eps, int32_t step, double lambda,
                                      uint8_t* mask_out, int64_t count, int64_t* popcount);

/* ------------------------------------------------------------------ adversary (lottery.hpp:36-42, 64-79) */
/* make_adversary (lottery.cpp:166-180): zero discriminator over m x D replay rows. */
MOSES_API int moses_adversary_create(const double* replay, int64_t m, int32_t D, int32_t width, double step_size,
                                     moses_adversary_t* out);
MOSES_API int moses_adversary_destroy(moses_adversary_t a);
MOSES_API int moses_adversary_get(moses_adversary_t a, double* weight, int32_t width, double* bias);
MOSES_API int moses_adversary_set(moses_adversary_t a, const double* weight, int32_t width, double bias);
/* adversarial_term (lottery.cpp:135-164) on explicit hidden activations (reference signature). */
MOSES_API int moses_adversarial_term(moses_adversary_t a, const double* hidden_source, int64_t ms,
                                     const double* hidden_target, int64_t nt, int32_t width, double beta,
                                     double* discriminator_loss, double* confusion);
/* tuner.cpp:252-256 fused: penultimate activations of the replay rows and the target rows under the
 * model's current params, then the discriminator step. */
MOSES_API int moses_adversarial_step(moses_adversary_t a, moses_model_t m, const double* target_features,
                                     int64_t n, int32_t D, double beta, double* discriminator_loss,
                                     double* confusion);
/* evolve (search.cpp:41-71) with the model scorer on the device: per generation the candidates are
 * encoded on the device from their enumeration indices and scored there; the GA's RngStream walk
 * (sample_config / mutate_config, KeyBuilder(seed, "evolve")) and the (score desc, config asc) sort
 * run on the host. SearchParams: population, generations, mutation_count, survivors, epsilon_random,
 * seed. Outputs (host): values_out (capacity x n_knobs), scores_out (capacity), n_out = final
 * population. m == NULL: linear test scorer sum_k lin_w[k] * value_k (double) instead of a model. */
MOSES_API int moses_evolve(moses_model_t m, const double* lin_w, const double* task4, const int64_t* domains,
                          const int32_t* domain_sizes, const int32_t* roles, int32_t n_knobs, int32_t population,
                          int32_t generations, int32_t mutation_count, int32_t survivors, double epsilon_random,
                          uint64_t seed, int64_t* values_out, double* scores_out, int64_t capacity, int64_t* n_out);
/* The Moses branch of a tuning step (tuner.cpp:251-262) in one call: moses_gradients(adv, beta) ->
 * moses_adversarial_step -> moses_lottery_step(mode, value, phase, alpha, lambda), bit-identical to
 * the three calls, with one host synchronisation; the discriminator step reuses the gradients'
 * forward pass over the same replay + batch rows. loss_out: the gradients' loss; dloss_out: the
 * discriminator loss before its step; popcount: transferable scalars. */
MOSES_API int moses_moses_step(moses_model_t m, moses_adversary_t adv, const double* features, const double* labels,
                              int64_t n, int32_t D, double beta, int32_t mode, double value, int32_t phase,
                              double alpha, double lambda, double* loss_out, double* dloss_out, int64_t* popcount);
/* discriminator_cross_entropy (lottery.cpp:207-218) */
MOSES_API int moses_discriminator_cross_entropy(const double* zs, int64_t m, const double* zt, int64_t n,
                                                double* out);

/* ------------------------------------------------------------------ candidate selection (search.cpp:32-37, 82-95) */
/* Indices of the k best scores ordered (score desc, index asc) — sort_desc's order when the
 * pool index is the lexicographic config order. k <= 4096. */
MOSES_API int moses_topk(const double* scores, int64_t n, int64_t k, int64_t* idx_out);
MOSES_API int moses_topk_device(const float* scores_dev, int64_t n, int64_t k, int64_t* idx_out_host);
/* select_batch (search.cpp:82-95) over a score-ordered candidate list: first k whose hash is
 * neither in `measured` nor already taken. Host-side. Returns the count written. */
MOSES_API int64_t moses_select_batch(const uint64_t* ordered_hashes, int64_t n, const uint64_t* measured,
                                     int64_t n_measured, int64_t batch_size, int64_t* out_positions);

/* ------------------------------------------------------------------ extensions */
/* Segment-sum pooling over CSR offsets on host buffers: out[p] = sum rows [off[p], off[p+1]). */
MOSES_API int moses_segment_sum(const double* h, int64_t rows, int32_t width, const int64_t* offsets,
                                int64_t programs, double* out);
/* Device variant (bf16 or f32 rows with row stride ld) -> fp32 out [programs][width]. */
MOSES_API int moses_segment_sum_device(const void* h_dev, int32_t dtype, int64_t ld, int32_t width,
                                       const int64_t* offsets_dev, int64_t programs, float* out_dev);
/* Biased MMD^2 with a Gaussian kernel between source and target representations. */
MOSES_API int moses_mmd2(const double* xs, int64_t m, const double* xt, int64_t n, int32_t width, double sigma,
                         double* out);
/* Same statistic over device-resident fp32 rows (stride ld floats): the cfg3 fine-tune path, where
   the source/target penultimate activations already live in HBM. tcgen05 kind::tf32 Gram tiles. */
MOSES_API int moses_mmd2_device(const float* xs, int64_t m, const float* xt, int64_t n, int32_t width, int64_t ld,
                                double sigma, double* out);

/* MMD^2 as a differentiable domain loss (north-star (4)): gradients() with beta * MMD^2(H_source, H_batch)
 * of the last hidden layer added to the objective, in the slot the reference's discriminator term uses
 * (model.cpp:215-238): `source` = ms source-domain rows (D wide; the replay rows), x / y the target batch.
 * loss_out = rank loss + beta * MMD^2. beta == 0 is gradients() bit for bit. Unpooled rows. */
MOSES_API int moses_gradients_mmd(moses_model_t m, const double* x, const double* y, int64_t n, int32_t D,
                                  const double* source, int64_t ms, double beta, double sigma, double* loss_out);
/* MMD^2 and d MMD^2 / d row for every source / target row (grad_s: m x width, grad_t: n x width, host). */
MOSES_API int moses_mmd2_grad(const double* xs, int64_t m, const double* xt, int64_t n, int32_t width, double sigma,
                              double* value, double* grad_s, double* grad_t);

/* ------------------------------------------------------------------ candidate generation */
/* Configurations [first, first+n) of a task's knob space in enumerate_configs order (space.cpp:168-191,
 * last knob fastest), on the device: encode_features rows (space.cpp:140-159; D >= 10 columns, entries
 * >= 10 zero, 1.0 at column D when ld > D) in dtype (F32 / BF16 / F64) with row stride ld, FNV-1a
 * config_hash values (space.cpp:193-197) and optionally the knob values (n x n_knobs). task4 =
 * {work_gflops, bytes_per_unit, ideal_log2_tiles, ideal_log2_unroll} (space.hpp:24-31); roles[i] =
 * template knob of knob i (0 tile_x, 1 tile_y, 2 unroll, 3 vectorize, 4 parallel, -1 other; knob_view
 * matches by name, space.cpp:123-138). Any output pointer may be NULL. Default stream. */
MOSES_API int moses_encode_configs_device(const double* task4, const int64_t* domains, const int32_t* domain_sizes,
                                         const int32_t* roles, int32_t n_knobs, uint64_t first, int64_t n,
                                         int32_t dtype, void* feat_dev, int64_t ld, int32_t D, uint64_t* hash_dev,
                                         int64_t* values_dev);
/* Host-output variant: float64 feature rows (n x 16) and hashes copied back (either may be NULL). */
MOSES_API int moses_encode_configs(const double* task4, const int64_t* domains, const int32_t* domain_sizes,
                                  const int32_t* roles, int32_t n_knobs, uint64_t first, int64_t n,
                                  double* features_out, uint64_t* hashes_out);

/* ------------------------------------------------------------------ simulated hardware */
/* device6 = {peak_gflops, parallel_units, vector_lanes, cache_bytes, measure_overhead_ms, noise_std}
 * (oracle.hpp DeviceSpec). Over configs [first, first+n) of the knob space (enumeration order as in
 * moses_encode_configs_device): clean_latency_ms (oracle.cpp:58-63) and measure() (oracle.cpp:65-88:
 * throughput with keyed Gaussian noise, latency, wall cost; label_dev = float throughput, the ranking
 * label). Any output may be NULL. Default stream. */
MOSES_API int moses_measure_configs_device(const double* device6, int32_t repeats, const char* device_id,
                                          const char* task_id, const double* task4, const int64_t* domains,
                                          const int32_t* domain_sizes, const int32_t* roles, int32_t n_knobs,
                                          uint64_t seed, uint64_t first, int64_t n, double* clean_ms_dev,
                                          double* throughput_dev, double* latency_dev, double* wall_cost_dev,
                                          float* label_dev);
/* true_best (oracle.cpp:90-105): exhaustive noise-free optimum on the device; the lexicographically
 * first configuration on exact ties. best_values (n_knobs) and best_latency are host outputs. */
MOSES_API int moses_true_best(const double* device6, const double* task4, const int64_t* domains,
                              const int32_t* domain_sizes, const int32_t* roles, int32_t n_knobs,
                              int64_t* best_values, double* best_latency);

/* ------------------------------------------------------------------ training-data pipeline */
/* generate_dataset (data.cpp:49-65) for ONE task: `samples` configurations drawn by
 * RngStream(KeyBuilder(seed, "gen", task_id)) through sample_config (space.cpp:94-100), their feature
 * rows (encode_features, packed layout as moses_encode_configs_device), knob values (samples x
 * n_knobs), and measure() outputs (oracle.cpp:65-88) — throughput / latency / wall cost in double,
 * label = float throughput. Any output may be NULL. A store over several tasks is the concatenation
 * in task order; its seq is the running row index (data.cpp:53-63). Default stream. */
MOSES_API int moses_generate_dataset_device(const double* device6, int32_t repeats, const char* device_id,
                                           const char* task_id, const double* task4, const int64_t* domains,
                                           const int32_t* domain_sizes, const int32_t* roles, int32_t n_knobs,
                                           int64_t samples, uint64_t seed, int32_t dtype, void* feat_dev, int64_t ld,
                                           int32_t D, int64_t* values_dev, double* throughput_dev,
                                           double* latency_dev, double* wall_cost_dev, float* label_dev);
/* encode_features over device rows of knob values (n x n_knobs int64): validate_config
 * (space.cpp:69-81) then the feature row. A value outside its domain fails with
 * MOSES_ERR_INVALID_CONFIG and *bad_row (host, may be NULL) = the first offending row. */
MOSES_API int moses_encode_values_device(const double* task4, const int64_t* domains, const int32_t* domain_sizes,
                                        const int32_t* roles, int32_t n_knobs, const int64_t* values_dev, int64_t n,
                                        int32_t dtype, void* feat_dev, int64_t ld, int32_t D, uint64_t* hash_dev,
                                        int64_t* bad_row);
/* pretrain's per-epoch seed KeyBuilder(seed, "epoch", epoch) (tuner.cpp:136-139). */
MOSES_API uint64_t moses_epoch_seed(uint64_t seed, uint64_t epoch);
/* make_ranking_batches (data.cpp:128-164) as a plan of row indices. record_task[i] indexes
 * task_ids (the ids the shuffle keys hash). Outputs (host, any may be NULL): rows_out (n_records),
 * batch_off (n_batches + 1 <= n_records / 2 + 1), batch_task (n_batches), n_batches, dropped
 * singleton chunks. Batch b covers rows_out[batch_off[b] .. batch_off[b+1]). */
MOSES_API int moses_ranking_plan(const int32_t* record_task, int64_t n_records, const char* const* task_ids,
                                int32_t n_task_ids, int32_t batch_size, uint64_t seed, int64_t* rows_out,
                                int64_t* batch_off, int32_t* batch_task, int64_t* n_batches, int64_t* dropped);
/* sample_replay_features' row choice (data.cpp:166-183): min(n_records, size) rows, no replacement. */
MOSES_API int moses_replay_rows(int64_t n_records, int64_t size, uint64_t seed, int64_t* rows_out, int64_t* n_out);
/* One pretrain epoch over a plan (tuner.cpp:140-155): for each batch in order, gather its rows of the
 * device-resident packed dataset (x_base rows of stride moses_packed_ld, labels y_base) -> gradients
 * -> momentum update. Plan arrays are host memory (moses_ranking_plan's output); mean_loss (host,
 * may be NULL) = mean of the per-batch losses (0 for an empty plan). Full-size batches replay one
 * CUDA graph (bf16 / tf32 handles). */
MOSES_API int moses_train_plan_device(moses_model_t m, const void* x_base, int64_t ldx, const float* y_base,
                                     int64_t n_records, const int64_t* rows, const int64_t* batch_off,
                                     int64_t n_batches, double learning_rate, double momentum, double* mean_loss);
/* pretrain (tuner.cpp:130-156) over a device-resident packed dataset: for each epoch e,
 * moses_ranking_plan(seed = moses_epoch_seed(seed, e)) then one momentum step per batch. The model
 * handle carries the initial parameters (the reference starts from init_random(dims, seed)). The host
 * computes epoch e+1's plan while the device runs epoch e. epoch_mean_loss (host, `epochs` entries)
 * and dropped_singletons (epoch 0, as PretrainLog) may be NULL. n_records == 0: MOSES_ERR_EMPTY_DATASET. */
MOSES_API int moses_pretrain_device(moses_model_t m, const void* x_base, int64_t ldx, const float* y_base,
                                   const int32_t* record_task, int64_t n_records, const char* const* task_ids,
                                   int32_t n_task_ids, int32_t batch_size, uint64_t seed, int32_t epochs,
                                   double learning_rate, double momentum, double* epoch_mean_loss,
                                   int64_t* dropped_singletons);
/* pretrain(store, tasks, hyper, log) (tuner.cpp:130-156) from host records: record_task[i] indexes
 * the task tables (task_ids, task4 = n_tasks x {work_gflops, bytes_per_unit, ideal_log2_tiles,
 * ideal_log2_unroll}; one knob template shared by all tasks, as the default task set); values are
 * n_records x n_knobs knob values, throughput the measured labels. The store is staged and encoded
 * on the device (grouped by task; batch composition unchanged), then moses_pretrain_device runs on
 * the handle, which carries the initial parameters. Invalid values fail with
 * MOSES_ERR_INVALID_CONFIG naming the record. */
MOSES_API int moses_pretrain(moses_model_t m, int32_t n_tasks, const char* const* task_ids, const double* task4,
                            const int64_t* domains, const int32_t* domain_sizes, const int32_t* roles,
                            int32_t n_knobs, const int32_t* record_task, const int64_t* values,
                            const double* throughput, int64_t n_records, int32_t batch_size, uint64_t seed,
                            int32_t epochs, double learning_rate, double momentum, double* epoch_mean_loss,
                            int64_t* dropped_singletons);
/* Job pool over independent pretrain runs sharing one device-resident dataset (the reference's
 * (strategy, seed) std::thread pool, tuner.cpp:57-69,331-374): job j runs moses_pretrain_device on
 * models[j] with seeds[j]; `threads` workers (0: MOSES_LAB_THREADS, else the hardware concurrency;
 * capped at n_jobs) claim jobs in order. Each handle has its own streams, so the jobs' latency-bound
 * steps overlap on the GPU. epoch_mean_loss: n_jobs x epochs (row per job); dropped_singletons:
 * n_jobs. Returns the lowest-numbered failing job's status. */
MOSES_API int moses_pretrain_jobs(int32_t n_jobs, const moses_model_t* models, const uint64_t* seeds,
                                 const void* x_base, int64_t ldx, const float* y_base, const int32_t* record_task,
                                 int64_t n_records, const char* const* task_ids, int32_t n_task_ids,
                                 int32_t batch_size, int32_t epochs, double learning_rate, double momentum,
                                 int32_t threads, double* epoch_mean_loss, int64_t* dropped_singletons);
/* The job grid across the GPUs of one process: job j runs on its handle's device
 * (recorded at moses_model_create) over that device's copy of the store, x_of[j] / y_of[j]. */
MOSES_API int moses_pretrain_jobs_mapped(int32_t n_jobs, const moses_model_t* models, const uint64_t* seeds,
                                        const void* const* x_of, int64_t ldx, const float* const* y_of,
                                        const int32_t* record_task, int64_t n_records, const char* const* task_ids,
                                        int32_t n_task_ids, int32_t batch_size, int32_t epochs, double learning_rate,
                                        double momentum, int32_t threads, double* epoch_mean_loss,
                                        int64_t* dropped_singletons);
/* ------------------------------------------------------------------ online tuning */
/* The tuner's per-task loop (tuner.cpp:158-286) and its (strategy, seed, task) job grid (tuner.cpp:307-374)
 * over this library's calls: per measured batch evolve (moses_evolve, device scoring) -> select_batch ->
 * measure (oracle.cpp:65-88 on the device) -> the controller's CV (controller.cpp:34-56, host) -> the
 * strategy's update (Moses: gradients with the replay adversary -> discriminator step -> lottery step;
 * vanilla / random-init: gradients -> apply_update), then the prediction-only tail. */
enum { MOSES_STRATEGY_RAW = 0, MOSES_STRATEGY_RANDOM_INIT = 1, MOSES_STRATEGY_PRETRAIN_ONLY = 2,
       MOSES_STRATEGY_VANILLA = 3, MOSES_STRATEGY_MOSES = 4 };               /* tuner.hpp StrategyKind */
typedef struct {                       /* oracle.hpp DeviceSpec */
  const char* id;
  double params[6];                    /* peak_gflops, parallel_units, vector_lanes, cache_bytes, measure_overhead_ms, noise_std */
  int32_t repeats;
} moses_device_spec;
typedef struct {                       /* space.hpp TaskSpec: task4 = {work_gflops, bytes_per_unit, ideal_log_tiles, ideal_log_unroll} */
  const char* id;
  double task4[4];
  const int64_t* domains;              /* concatenated knob domains (strictly increasing each) */
  const int32_t* domain_sizes;
  const int32_t* roles;
  int32_t n_knobs;
} moses_task_spec;
typedef struct {                       /* tuner.hpp TuneBudget (search seed ignored: per-batch streams) */
  int32_t trials_per_task;
  double train_fraction;
  int32_t num_batches;
  double cv_threshold;
  int32_t population, generations, mutation_count, survivors;   /* search.hpp SearchParams */
  double epsilon_random;
  double learning_rate, weight_decay, adversary_beta;           /* model.hpp TrainHyper */
  int32_t lottery_mode;                /* MOSES_MODE_THRESHOLD / MOSES_MODE_RATIO */
  double lottery_value;
  int32_t adversary;                   /* Moses only */
  int32_t replay_size;
} moses_tune_budget;
typedef struct {                       /* tuner.hpp TaskResult + ControllerTrace; caller-owned arrays */
  int64_t capacity;                    /* rows of values / throughput / latency / wall_cost / predicted_scores */
  int64_t* values;                     /* [capacity x n_knobs] measured configurations, measurement order */
  double* throughput;
  double* latency;
  double* wall_cost;
  int64_t n_records;
  int64_t* best_values;                /* [n_knobs] */
  double best_latency_ms;
  double wall_cost_ms;
  double* batch_means;                 /* [num_batches] */
  double* cvs;                         /* [num_batches]; NaN where fewer than two means existed */
  int32_t n_batch_means;
  int32_t termination_batch, measured_trials, prediction_trials, unspent_trials;
  double* predicted_scores;            /* [capacity] prediction-only tail */
} moses_task_result;
/* tune_task on the parameters held by `m` (updated in place: pass a copy per job, tuner.cpp:349).
 * source_features: the source store's encoded rows (n_source x dims[0], store order), needed by Moses with
 * the adversary on (the replay buffer, data.cpp:166-183); NULL otherwise. */
MOSES_API int moses_tune_task(moses_model_t m, int32_t strategy, const moses_device_spec* device,
                              const moses_task_spec* task, const moses_tune_budget* budget, uint64_t seed,
                              const double* source_features, int64_t n_source, moses_task_result* out);
/* The job grid: job j = (strategies[j], seeds[j], tasks[task_of[j]]) on handle models[j] (a per-job copy,
 * on any GPU of the process), claimed in order by `threads` workers (0: one per job, capped at 64), the
 * first failing job's status returned. results[j] as moses_tune_task's out. */
MOSES_API int moses_tune_jobs(int32_t n_jobs, const moses_model_t* models, const int32_t* strategies,
                              const uint64_t* seeds, const int32_t* task_of, const moses_task_spec* tasks,
                              int32_t n_tasks, const moses_device_spec* device, const moses_tune_budget* budget,
                              const double* source_features, int64_t n_source, int32_t threads,
                              moses_task_result* results);

/* Line-delimited record files (data.cpp:67-126). moses_records_read fails with MOSES_ERR_IO,
 * MOSES_ERR_PARSE (message names "<path>:line N") or MOSES_ERR_MISSING_FIELD. */
MOSES_API int moses_records_create(moses_records_t* out);
MOSES_API int moses_records_read(const char* path, moses_records_t* out);
MOSES_API void moses_records_destroy(moses_records_t r);
/* append n records of one task / device, n_values knob values each (values: n x n_values) */
MOSES_API int moses_records_append(moses_records_t r, const char* task_id, const char* device_id, int64_t n,
                                  int32_t n_values, const int64_t* values, const double* throughput,
                                  const double* latency, const double* wall_cost, const uint64_t* seq);
MOSES_API int moses_records_write(moses_records_t r, const char* path);
MOSES_API int moses_records_shape(moses_records_t r, int64_t* n_records, int64_t* n_values, int32_t* n_tasks,
                                 int32_t* n_devices);
/* interned ids in first-appearance order; NULL when out of range */
MOSES_API const char* moses_records_task_id(moses_records_t r, int32_t t);
MOSES_API const char* moses_records_device_id(moses_records_t r, int32_t d);
/* flat copies into caller buffers (pinned host memory for a following upload); any may be NULL.
 * value_off: n_records + 1 offsets into values. */
MOSES_API int moses_records_export(moses_records_t r, int32_t* task_index, int32_t* device_index, int64_t* value_off,
                                  int64_t* values, double* throughput, double* latency, double* wall_cost,
                                  uint64_t* seq);
/* Test hook: force the fused ranking step's grid form (1) instead of the default policy (0:
 * 16-CTA cluster form when the batch fits it, else the symmetric form, else the grid form). */
MOSES_API int moses_debug_set_rank_grid(int32_t on);
/* Test hook: allow (1, default) or disable (0) the ranking step's symmetric form (each pair once). */
MOSES_API int moses_debug_set_rank_sym(int32_t on);
/* Test hooks: split-bf16 weight gradients split over the batch rows in clusters (1, default) or one
 * CTA per tile (0); splits > 0 forces the cluster width. Probe: TMEM promotion interval in 64-row
 * k-blocks (0 = default) and an optional device buffer of clock64 / globaltimer stamps. */
MOSES_API int moses_debug_set_wgrad_sk(int on, int splits);
MOSES_API int moses_debug_wgrad_sk_probe(int kc, void* trace);
/* Test hook: run the last hidden level's split-bf16 weight gradient beside the dZ chain (1, default). */
MOSES_API int moses_debug_set_wgrad_early(int on);
/* Test hook: split-bf16 fused chain on CTA pairs (1) or single CTAs (0, default); bit-identical results. */
MOSES_API int moses_debug_set_chain_pair(int on);
/* Test hook: force the sequential sampling walk in moses_generate_dataset_device. */
MOSES_API int moses_debug_force_serial_sampling(int32_t on);

/* ------------------------------------------------------------------ synthetic TenSet-shaped data (bench) */
/* Rows [row0, row0+n) of the keyed SplitMix64 generator, written in the packed layout. */
MOSES_API int moses_synth_features_device(uint64_t seed, int64_t row0, int64_t n, int32_t D, int32_t dtype,
                                          void* dst, int64_t ld);
MOSES_API int moses_synth_labels_device(uint64_t seed, int64_t row0, int64_t n, float* dst);
/* CSR offsets of `programs` programs with 1 + below(max_stmts) statements each (host). */
MOSES_API int moses_synth_offsets(uint64_t seed, int64_t programs, int32_t max_stmts, int64_t* offsets);

/* ------------------------------------------------------------------ multi-GPU
 * NCCL communicators behind the ABI (NCCL is loaded at run time: libnccl.so.2). Either one process per
 * GPU (rank 0 makes the id with moses_comm_unique_id, the caller distributes its 128 bytes, every rank
 * calls moses_comm_init_rank on its current device) or one process for n GPUs (moses_comm_init_all:
 * ncclCommInitAll, comms_out[i] drives devices[i]). */
typedef struct moses_comm* moses_comm_t;
MOSES_API int moses_comm_unique_id(uint8_t* id_out, int64_t cap);
MOSES_API int moses_comm_init_rank(const uint8_t* id, int32_t nranks, int32_t rank, moses_comm_t* out);
MOSES_API int moses_comm_init_all(int32_t ndev, const int32_t* devices, moses_comm_t* comms_out);
MOSES_API int moses_comm_destroy(moses_comm_t c);
MOSES_API int moses_comm_info(moses_comm_t c, int32_t* nranks, int32_t* rank, int32_t* device);
/* Data-parallel training on a handle (tuner.cpp:134-154's batch loop across ranks). mode 0: none;
 * 1: throughput mode, every rank steps its own batch and the gradients are averaged (ncclAvg) before the
 * update; 2: exact batch, the global batch is the rank-ordered concatenation of every rank's rows: local
 * forward, all-gather of scores + labels, pair terms of the local rows against the whole batch
 * (model.cpp:71-106, each distinct-label pair counted once), all-reduce of (loss, pairs), local backward,
 * all-reduce (sum) of the gradients = the gradient of the global batch up to summation order. Mode 2
 * takes unpooled rows. With a communicator set, moses_train_graph_create[_pooled] capture the
 * collectives and the update into the step graph. */
MOSES_API int moses_model_set_comm(moses_model_t m, moses_comm_t c, int32_t mode);
MOSES_API int moses_dp_allreduce_gradients(moses_model_t m, int32_t average);
/* one data-parallel step on device rows (packed layout, moses_packed_ld; fp32 labels); loss_out: the
 * rank's batch loss (mode 1) or the global batch loss (mode 2) */
MOSES_API int moses_dp_train_step(moses_model_t m, const void* x_dev, int64_t ldx, const float* y_dev, int64_t n,
                                  double learning_rate, double momentum, double* loss_out);
/* the exact-batch step's phases around its collectives (tests; callers with their own transport):
 * forward writes the n local scores / labels to s_slot / y_slot (device); rank takes the gathered
 * n_global scores / labels and this rank's offset p0, writes (loss sum, pair count) partials to
 * totals_dev[2]; backward takes the summed totals and leaves this rank's gradient share on the handle. */
MOSES_API int moses_dp_exact_forward(moses_model_t m, const void* x_dev, int64_t ldx, const float* y_dev, int64_t n,
                                     float* s_slot, float* y_slot);
MOSES_API int moses_dp_exact_rank(moses_model_t m, const float* s_global, const float* y_global, int64_t n_global,
                                  int64_t p0, double* totals_dev);
MOSES_API int moses_dp_exact_backward(moses_model_t m, int64_t n_global, const double* totals_dev, double* loss_out);
/* Sharded candidate scoring (cfg4): top-k of this rank's shard [row0, row0 + n_local) of the pool, winners
 * all-gathered and merged by (score desc, index asc) (search.cpp:32-37); idx_out[k] (host) is the same on
 * every rank and equals the single-device top-k of the whole pool. */
MOSES_API int moses_topk_sharded(moses_comm_t c, const float* scores_dev, int64_t n_local, int64_t row0, int64_t k,
                                 int64_t* idx_out);

/* ------------------------------------------------------------------ files (model.cpp:344-412, lottery.cpp:182-240) */
MOSES_API int64_t moses_serialize(const int32_t* dims, int32_t ndims, const double* params, const double* momentum,
                                  uint8_t* out, int64_t cap);
MOSES_API int moses_deserialize(const uint8_t* bytes, int64_t len, int32_t* dims_out, double* params,
                                double* momentum, int64_t cap);
MOSES_API int64_t moses_write_mask(const uint8_t* mask, int64_t n, int32_t phase, int32_t mode, double value,
                                   uint8_t* out, int64_t cap);
MOSES_API int moses_read_mask(const uint8_t* bytes, int64_t len, uint8_t* mask_out, int64_t cap, int64_t* n,
                              int32_t* phase, int32_t* mode, double* value);

/* ------------------------------------------------------------------ timing helpers (bench) */
/* Calling thread: make moses_apply_update asynchronous on the handle's stream (device-resident loops). */
MOSES_API int moses_set_async(int32_t on);
/* Device-time attribution: CUDA-event brackets per kernel class between begin and end.
 * Classes: 0 gemm_fwd, 1 gemm_dgrad, 2 gemm_wgrad, 3 rank, 4 head, 5 update, 6 select, 7 topk, 8 other. */
MOSES_API int moses_profile_begin(void);
MOSES_API int moses_profile_end(double* ms_by_cat, int64_t* count_by_cat, int32_t ncat);
/* Raw pointers into the handle (device): params fp32, gradients fp32, momentum fp32. */
MOSES_API int moses_model_device_ptrs(moses_model_t m, float** params, float** grads, float** momentum);
MOSES_API int moses_model_stream(moses_model_t m, void** stream);
/* Test hook: one raw tcgen05 GEMM C = A * B^T on device buffers (elem 2 = bf16, 4 = tf32;
 * epi 0 = bias/ReLU store, 1 = ReLU'-masked store, 2 = fp32 store; bn 0 = auto). */
MOSES_API int moses_debug_gemm(int elem, int M, int N, int K, const void* A, long long lda, int a_mn, const void* B,
                               long long ldb, int b_mn, int epi, void* out, long long ldo, const float* bias, int relu,
                               int bn, const void* mask, long long ldm);

#ifdef __cplusplus
}
#endif
#endif /* MOSES_GPU_H_ */
