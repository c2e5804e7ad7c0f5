/* rhino_exec.h — C-ABI of the B200-native executor for Rhino-partitioned tensor programs.
 *
 * The reference (arXiv 2302.08141, /root/reference/proj) is a planner only: it emits an
 * ExecutionPlan (proj/include/parashard/planner.h:69-84) whose per-op, per-mesh-axis
 * AxisSpec (proj/include/parashard/sharding.h:32-53) fixes how every tensor is placed, and whose
 * OpStrategy (sharding.h:99-111) fixes what each op demands of its inputs.  It has no executor
 * (SPEC.md:17, :482).  This header is the drop-in execution boundary a maintainer binds from the
 * reference's C++ host code: the `parashard` CLI's RunPlan tail (proj/tools/parashard_main.cpp:77-81)
 * lowers plan + strategies into rh_op records (see paper_2302_08141_b200/host/rh_lower.h) and calls
 * rh_program_load / rh_program_run.  Plain C types only: no torch, no C++ across the ABI.
 *
 * Conventions:
 *   - every function returns 0 on success and a negative rh_status otherwise; rh_last_error()
 *     returns the thread-local message of the last failure.  No C++ exception crosses the ABI.
 *   - handles are opaque and owned by the library; the caller owns host buffers.
 *   - calls are synchronous from the host's view; device timing uses CUDA events.
 *   - global rank = sum_k coord_k * prod_{j>k} dims_j (row-major, axis 0 slowest), matching
 *     the planner's grid.dims = {machines, gpus_per_machine} (proj/src/planner.cpp:58-63).
 */
#ifndef RHINO_EXEC_H_
#define RHINO_EXEC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RH_MAX_RANK 8
#define RH_MAX_AXES 4
#define RH_UID_BYTES 128

typedef enum {
  RH_OK = 0,
  RH_ERR_INVALID = -1,     /* bad argument / unsupported program (message says which) */
  RH_ERR_CUDA = -2,        /* CUDA runtime failure */
  RH_ERR_NCCL = -3,        /* NCCL failure */
  RH_ERR_STATE = -4,       /* call out of order */
  RH_ERR_UNSUPPORTED = -5, /* valid per the reference, not executable by this build */
  RH_ERR_TIMEOUT = -6      /* a cross-GPU barrier did not complete within RH_SYNC_TIMEOUT_MS
                              (default 60 s): a peer died or the schedules diverged */
} rh_status;

/* parashard::AxisSpec::Kind (sharding.h:33) — note the reference enum order is
 * {kShard, kReplicated, kPartial}. */
typedef enum { RH_SHARD = 0, RH_REPLICATED = 1, RH_PARTIAL = 2 } rh_spec_kind;

typedef struct {
  int32_t kind;    /* rh_spec_kind */
  int32_t dim;     /* RH_SHARD only */
  int64_t stride;  /* RH_SHARD only: block-cyclic block length along `dim` */
} rh_spec;

/* parashard::OpKind, same order (proj/include/parashard/ir.h:58-70). */
typedef enum {
  RH_OP_PARAMETER = 0,
  RH_OP_INPUT = 1,
  RH_OP_MATMUL = 2,
  RH_OP_ADD = 3,
  RH_OP_MUL = 4,
  RH_OP_UNARY = 5,
  RH_OP_RESHAPE = 6,
  RH_OP_TRANSPOSE = 7,
  RH_OP_REDUCE_SUM = 8,
  RH_OP_BROADCAST = 9,
  RH_OP_CONCAT = 10
} rh_op_kind;

/* UnaryElementwise `fn` labels (proj/src/ir.cpp:83-85).  The reference calls the label
 * "informational" (ir.h:87); DESIGN.md §Semantics fixes what each one computes. */
typedef enum {
  RH_FN_UNLABELED = 0, /* fixture chains carry no fn (proj/src/fixtures.cpp:60): tanh by default */
  RH_FN_RELU = 1,
  RH_FN_GELU = 2,
  RH_FN_TANH = 3,
  RH_FN_EXP = 4,
  RH_FN_SIGMOID = 5,
  RH_FN_SOFTMAX = 6,   /* row softmax over the last dim; last dim must be unsharded */
  RH_FN_NEG = 7,
  RH_FN_RSQRT = 8,     /* 1/sqrt(|x| + 1e-6) */
  RH_FN_IDENTITY = 9
} rh_unary_fn;

/* The IR carries only elem_bytes (ir.h:37-56); the dtype is this side channel. */
typedef enum { RH_F32 = 0, RH_BF16 = 1 } rh_dtype;

/* One lowered operator: the reference Operator (ir.h:72-95) plus, per mesh axis, the
 * OpStrategy the planner chose for it (sharding.h:99-111): out_spec = output_spec and
 * in_specs[axis * n_in + slot] = input_specs[slot]. */
typedef struct {
  int32_t kind;                  /* rh_op_kind */
  int32_t fn;                    /* rh_unary_fn (RH_OP_UNARY only) */
  int32_t dtype;                 /* rh_dtype */
  int32_t rank;
  int64_t dims[RH_MAX_RANK];     /* global output shape */
  int32_t n_in;
  const int32_t* inputs;         /* n_in producer op indices */
  int32_t transpose_a, transpose_b; /* MatMul */
  int32_t axis;                  /* ReduceSum / Concat */
  int32_t has_perm;              /* Transpose: 0 = reverse all axes (sharding.cpp:173-180) */
  int32_t perm[RH_MAX_RANK];
  rh_spec out_spec[RH_MAX_AXES];
  const rh_spec* in_specs;       /* [n_axes][n_in], axis-major */
  /* Pipeline programs only (rh_program_load_pipeline; ignored by rh_program_load): the stage
   * that computes the op (ExecutionPlan.stages.stage_of, planner.h:69-84), its microbatch
   * (1..m) and its task in the stage's 1F1B order (proj/src/taskgraph.cpp:173-211):
   * RH_PHASE_FWD / RH_PHASE_BWD / RH_PHASE_ACC (LocalAccumulate, taskgraph.cpp:149-160). */
  int32_t stage;
  int32_t microbatch;
  int32_t phase;
} rh_op;

#define RH_PHASE_FWD 0
#define RH_PHASE_BWD 1
#define RH_PHASE_ACC 2

/* rh_program_load flags */
#define RH_FLAG_UNLABELED_IDENTITY 0x1u /* unlabeled unary = identity instead of tanh */
#define RH_FLAG_NO_FUSION 0x2u          /* materialize every op (no chain / epilogue fusion) */
#define RH_FLAG_TRANSPORT_NCCL 0x4u     /* resharding through NCCL collectives + pack kernels
                                           (baseline) instead of the peer-memory kernels */
#define RH_FLAG_NO_MATERIALIZE 0x8u     /* leave program outputs in their planned spec */
#define RH_FLAG_SIMT_GEMM 0x10u         /* force the CUDA-core GEMM (test/reference kernel) */
#define RH_FLAG_NO_GRAPH 0x20u          /* launch eagerly instead of replaying a CUDA graph */
#define RH_FLAG_REDUCE_OUTPUTS 0x80u    /* outputs: reduce Partial axes only (P -> R), leave
                                           sharded axes sharded (a training step's gradients) */
#define RH_FLAG_NO_OVERLAP 0x100u       /* dist: keep every transition on the main stream (no
                                           side-stream overlap of off-critical-path transitions) */
#define RH_FLAG_NO_PDL 0x200u          /* no programmatic dependent launch between compute kernels */
#define RH_FLAG_KEEP_ALL 0x40u          /* give every intermediate its own buffer (no arena reuse)
                                           so rh_program_read_* can read any op after a run */

typedef struct rh_runtime rh_runtime;
typedef struct rh_mesh rh_mesh;
typedef struct rh_program rh_program;

const char* rh_last_error(void);
const char* rh_version(void);

/* NCCL unique id for rh_runtime_create_dist (rank 0 creates, the caller broadcasts it). */
int rh_get_unique_id(uint8_t uid[RH_UID_BYTES]);

/* Single process, `n_ranks` logical ranks; rank i runs on CUDA device cuda_ids[i].  Ids may
 * repeat: several logical ranks then share one GPU (emulated mesh, collectives run as one
 * kernel over all ranks' buffers). */
int rh_runtime_create(int n_ranks, const int* cuda_ids, rh_runtime** out);
/* One process per GPU (torchrun): this process is `rank` of `world` on device `cuda_id`.
 * Peer buffers are mapped over NVLink with CUDA IPC; NCCL carries the bootstrap and the
 * RH_FLAG_TRANSPORT_NCCL baseline. */
int rh_runtime_create_dist(int world, int rank, int cuda_id, const uint8_t uid[RH_UID_BYTES],
                           rh_runtime** out);
int rh_runtime_world(const rh_runtime* rt, int* world, int* first_local_rank, int* n_local);
void rh_runtime_destroy(rh_runtime* rt);

/* Device mesh (parashard::DeviceMesh::dims, mesh.h:44-57); prod(dims) == world. */
int rh_mesh_create(rh_runtime* rt, int n_axes, const int* dims, rh_mesh** out);
void rh_mesh_destroy(rh_mesh* mesh);

/* A pipeline-parallel program (ExecutionPlan.pipeline_axis >= 0): mesh axis `pipeline_axis`
 * holds the S stages (every spec Replicated on it); a rank with pipeline coordinate s runs only
 * the ops of stage s, SPMD over the other axes; a value consumed by a later (or earlier) stage
 * moves between the two ranks with equal non-pipeline coordinates (Send/Recv, taskgraph.cpp:
 * 115-130) and is then resharded within the receiving stage (cut placeholders, planner.cpp:
 * 84-91).  Each stage runs its tasks in 1F1B order (taskgraph.cpp:173-211).  `apply` (n_apply
 * pairs {gradient op, parameter op}, may be 0): after the step, every parameter is updated in
 * place, p -= lr * g (ApplyGradients, taskgraph.cpp:161-165), by its stage. */
int rh_program_load_pipeline(rh_mesh* mesh, int pipeline_axis, const rh_op* ops, int n_ops, const int* outputs,
                             int n_out, const int* apply, int n_apply, float lr, uint32_t flags,
                             rh_program** out);

/* Lower + allocate a partitioned program.  `outputs` are the program outputs
 * (TensorProgram::output_indices, ir.cpp:321-330); unless RH_FLAG_NO_MATERIALIZE they are
 * materialized Replicated at the end of every run (final AllReduce / AllGather). */
int rh_program_load(rh_mesh* mesh, const rh_op* ops, int n_ops, const int* outputs, int n_out,
                    uint32_t flags, rh_program** out);
void rh_program_destroy(rh_program* prog);

/* Synthetic sources: Philox4x32-10 keyed by (seed, op index, global flat index); inputs
 * U[-1,1), parameters U[-1,1)*sqrt(3/dims[0]); bf16 by round-to-nearest-even. */
int rh_program_init_synthetic(rh_program* prog, uint64_t seed);
/* Host full tensor of a source op -> every local rank's shard (H2D + on-device slice). */
int rh_program_write_full(rh_program* prog, int op, const void* src, size_t bytes);
/* Run the program `iters` times; *ms_per_iter = device time per run (max over local ranks). */
int rh_program_run(rh_program* prog, int iters, double* ms_per_iter);
/* End-to-end step through host buffers: H2D of every `n_in` (op, host ptr) input, one run,
 * D2H of the first n_outs program outputs into out_ptrs: the full tensor when materialized
 * (in a multi-process run: this process's 1/world contiguous slice of it, at its offset in
 * out_ptrs, so the processes' slices together are the full tensor), else this process's
 * first local rank's shard (rh_program_local_bytes).  Timed inside. */
int rh_program_step_host(rh_program* prog, int n_in, const int* in_ops, const void* const* in_ptrs,
                         int n_outs, void* const* out_ptrs, double* ms);

/* Pipelined end-to-end steps (one local rank per process): `iters` steps, each with the H2D of
 * every input and the D2H of the first n_outs outputs (as rh_program_step_host), step i's H2D
 * overlapping step i-1's run and step i-2's D2H through double-buffered device stages;
 * *ms_per_iter = time from before the first H2D to after the last D2H, divided by iters. */
int rh_program_run_host(rh_program* prog, int iters, int n_in, const int* in_ops, const void* const* in_ptrs,
                        int n_outs, void* const* out_ptrs, double* ms_per_iter);

/* Local buffer of `op` on global `rank` (must be local to this process); bytes must equal the
 * local size.  Returns the buffer as laid out on the device (block-cyclic local order). */
int rh_program_read_local(rh_program* prog, int op, int rank, void* dst, size_t bytes);
/* Full tensor of `op`: program outputs read the materialized buffer; other ops are assembled
 * from the local shards (every rank must be local). */
int rh_program_read_full(rh_program* prog, int op, void* dst, size_t bytes);
int rh_program_local_bytes(const rh_program* prog, int op, int rank, size_t* bytes);
/* Device memory of the program per rank: the whole symmetric arena, and the part of it that is
 * persistent (sources, outputs, peer-read transition sources, tables, scratch); the rest is the
 * liveness-planned pool that intermediates share (none with RH_FLAG_KEEP_ALL). */
int rh_program_memory(const rh_program* prog, size_t* arena_bytes, size_t* pool_bytes);
/* Verification: the full value of the tensor `op` consumed at input `slot` (its producer in the
 * layout the op's strategy demanded, after resharding), assembled from every rank (all local). */
int rh_program_read_input_full(rh_program* prog, int op, int slot, void* dst, size_t bytes);

/* Schedule introspection: one record per scheduled step (kernel or collective). */
typedef struct {
  char name[64];        /* e.g. "matmul b00_q", "reshard all_to_all ctx" */
  int32_t kind;         /* 0 kernel, 1 transition, 2 barrier/sync */
  int32_t launches;     /* kernels this step launches per run on one rank */
  double alg_bytes;     /* algorithmic HBM bytes per rank per run (read + write) */
  double alg_flops;     /* algorithmic flops per rank per run */
  double wire_bytes;    /* reshard_cost bytes (sharding.cpp:104-142) per rank, 0 if local */
  double ms;            /* mean device time per run from the last rh_program_profile */
} rh_step_info;
int rh_program_num_steps(const rh_program* prog, int* n);
int rh_program_step_info(const rh_program* prog, int i, rh_step_info* out);
/* Run `iters` times with CUDA events around every step on the step's stream (rank 0 of this
 * process); fills rh_step_info.ms. */
int rh_program_profile(rh_program* prog, int iters, double* ms_per_iter);
/* Kernel launches per run summed over this process's ranks. */
int rh_program_launch_count(const rh_program* prog, int64_t* launches);

/* The executor's local-op rule table on its own (host only, no device): the output spec per mesh
 * axis that op `op`'s local computation produces when its inputs arrive in the specs its
 * strategy demands (ops[op].in_specs) — the local side of FollowInput / ProduceOutput
 * (proj/src/sharding.cpp:225-388), composed over axes as EffectiveShapes does (:390-403).  A
 * planned out_spec that differs from it is executed by the pin fallback (compute, then slice,
 * sharding.cpp:477-487).  Fails (RH_ERR_INVALID) when no local rule exists. */
int rh_op_natural_specs(const rh_op* ops, int n_ops, int op, int n_axes, const int* mesh_dims, rh_spec* out);

/* Microbenchmark entry (config C4): one transition `from -> to` on mesh axis `axis` of a
 * tensor of global shape dims (dtype), src/dst = device buffers of every LOCAL rank (in local
 * rank order).  `iters` back-to-back repetitions, *ms = mean device time (max over ranks). */
int rh_reshard(rh_mesh* mesh, int axis, rh_spec from, rh_spec to, int ndim, const int64_t* dims,
               int dtype, void* const* src, void* const* dst, uint32_t flags, int iters, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* RHINO_EXEC_H_ */
