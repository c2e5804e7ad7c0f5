/* ref_cpu_exec.h — CPU ORACLE for partitioned-program execution.  TEST INFRASTRUCTURE ONLY:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it, and only as the checker or the timed CPU baseline — never as the product path.
 *
 * The reference (Rhino, /root/reference/proj) has no executor, so "the
 * reference's own CPU execution" of a partitioned program is this restatement of its semantics:
 *   op meaning            proj/src/ir.cpp:90-243 (InferOutputShape / OperatorFlops)
 *   spec validity/layout  proj/src/sharding.cpp:47-72 (SpecValidForShape, LocalShape, OwnerOfFlatIndex)
 *   per-op local rules    proj/src/sharding.cpp:225-388 (FollowInput / ProduceOutput)
 *   pin fallback          proj/src/sharding.cpp:477-487 (compute replicated, slice locally)
 *   transitions           proj/src/sharding.cpp:104-142, include/parashard/sharding.h:76-85
 *   axis composition      proj/src/sharding.cpp:390-403 (EffectiveShapes)
 *   execution order       proj/src/ir.cpp:381-412 (TopoOrderIndices)
 * Numeric parity is UNPINNED by the reference (no golden vectors; fn labels informational,
 * ir.h:87): the semantics fixed in DESIGN.md §Semantics are the pin, and placement is pinned by
 * the SPEC.md worked examples (tests/test_oracle.py).
 *
 * It runs a lowered program (rh_op records, include/rhino_exec.h) two ways:
 *   - unpartitioned: one device, full tensors (the single-device result);
 *   - partitioned: all world ranks simulated, each op on its block-cyclic local buffers, every
 *     resharding edge realised by assembling the global value and re-slicing it (no per-axis
 *     collective decomposition: deliberately independent of the GPU executor's algorithm).
 */
#ifndef REF_CPU_EXEC_H_
#define REF_CPU_EXEC_H_

#include <stddef.h>
#include <stdint.h>

#include "rhino_exec.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ox_program ox_program;

const char* ox_last_error(void);

/* Philox4x32-10 (Salmon et al., SC'11) on one (counter, key) block. */
void ox_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* The synthetic value of global element `flat` of op `op_index` (see rhino_exec.h). */
float ox_synthetic_value(uint64_t seed, uint32_t op_index, uint64_t flat, int is_param,
                         int64_t fan_in);
uint16_t ox_f32_to_bf16(float x);
float ox_bf16_to_f32(uint16_t x);

/* SPEC-level layout primitives (sharding.cpp:47-72 + the implied local coordinate). */
int64_t ox_owner_of_flat(int ndim, const int64_t* dims, rh_spec spec, int d, int64_t flat);
int64_t ox_local_of_flat(int ndim, const int64_t* dims, rh_spec spec, int d, int64_t flat);

/* One single-axis transition over a group of d ranks on a tensor of global shape dims:
 * src[r] holds rank r's buffer in `from`, dst[r] receives rank r's buffer in `to`.
 * Partial sums are accumulated in rank order 0..d-1 in fp32 (bf16: rounded once). */
int ox_reshard(int d, int ndim, const int64_t* dims, rh_spec from, rh_spec to, int dtype,
               const void* const* src, void* const* dst);

int ox_load(const rh_op* ops, int n_ops, const int* outputs, int n_out, int n_axes,
            const int* mesh, uint32_t flags, ox_program** out);
void ox_destroy(ox_program* p);
int ox_init_synthetic(ox_program* p, uint64_t seed);
/* Overrides a source op's value (full tensor in its dtype). */
int ox_set_full(ox_program* p, int op, const void* src, size_t bytes);
/* threads <= 0: all OpenMP threads. */
int ox_run_unpartitioned(ox_program* p, int threads);
int ox_run_partitioned(ox_program* p, int threads);
/* which = 0: unpartitioned result; 1: assembled from the partitioned local buffers. */
int ox_read_full(ox_program* p, int op, int which, void* dst, size_t bytes);
int ox_read_local(ox_program* p, int op, int rank, void* dst, size_t bytes);
int ox_local_bytes(ox_program* p, int op, size_t* bytes);
/* Flops of the last run (unpartitioned: sum; partitioned: per rank max). */
double ox_last_flops(ox_program* p);

#ifdef __cplusplus
}
#endif
#endif
