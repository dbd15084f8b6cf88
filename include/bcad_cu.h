/*
 * bcad_cu.h — C-ABI of the B200-native mixed-mode broadcast differentiation
 * library (libbcad_cu.so). Plain pointers and sizes only: no CUDA, torch or
 * C++ types cross this boundary (streams are opaque `void*` cudaStream_t,
 * NULL = the legacy default stream).
 *
 * This is the boundary the reference's hot path crosses when its host C++
 * API (the include/bcad headers of this repo, mirroring /root/reference/proj/
 * include/bcad) is backed by the GPU. Every entry point names the reference
 * interface it replaces:
 *
 *   bcad_cu_kernel_lookup  <- BroadcastKernel<Real>(n, m, name, body)
 *                             proj/include/bcad/kernel.hpp:26-36
 *   bcad_cu_broadcast_shape<- broadcast_shape / make_broadcast_plan
 *                             proj/include/bcad/shape.hpp:70-90, broadcast.hpp:25-41
 *   bcad_cu_forward        <- broadcast_diag_jacobian(kernel, args, want_primal)
 *                             proj/include/bcad/forward.hpp:98-150 (partials != NULL)
 *                             broadcast_apply(kernel, args)
 *                             proj/include/bcad/broadcast.hpp:102-125 (partials == NULL)
 *   bcad_cu_pullback       <- the CacheForward backward of mixed_broadcast:
 *                             backprop_diag + tensor_zip + accumulate_adjoint/scatter_add
 *                             proj/include/bcad/mixed.hpp:27-41, 68-72,
 *                             broadcast.hpp:174-183, 210-217, tape.hpp:179-183
 *                             and, with partials == NULL, the RecomputeReverse
 *                             backward (mixed.hpp:82-89) fused into one pass.
 *   bcad_cu_scatter_add    <- Tape::accumulate_adjoint / scatter_add
 *                             proj/include/bcad/tape.hpp:179-183, broadcast.hpp:210-217
 *   bcad_cu_allreduce_adjoints  (new; the reference is single-process) — NCCL
 *                             sum of batch-broadcast argument adjoints.
 *
 * Status codes map one-to-one onto proj/include/bcad/errors.hpp:8-66.
 * Ownership: the caller allocates every buffer (device memory may come from
 * bcad_cu_malloc); the library never retains a pointer after return. The
 * only library-owned device state is a per-device pool of 8-byte error
 * words, one taken by each in-flight call of a may-raise kernel.
 * Thread safety: reentrant; concurrent calls on different streams or host
 * threads do not share state. A may-raise kernel (bcad_cu_kernel_may_raise)
 * synchronises its stream after the launch to decode the domain check
 * (forward.hpp:137-146) and refuses CUDA-graph capture with
 * BCAD_CU_ERR_CONFIG; every other launch is asynchronous and capturable.
 */
#ifndef BCAD_CU_H
#define BCAD_CU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BCAD_CU_MAX_RANK 8
#define BCAD_CU_MAX_INPUTS 32  /* kMaxKernelInputs, kernel.hpp:14 */
#define BCAD_CU_MAX_OUTPUTS 8  /* kMaxKernelOutputs, kernel.hpp:15 */
#define BCAD_CU_VERSION 1

typedef enum bcad_cu_status {
    BCAD_CU_OK = 0,
    BCAD_CU_ERR_TAG_MISMATCH = 1,        /* TagMismatch            errors.hpp:14 */
    BCAD_CU_ERR_DIVISION_BY_ZERO = 2,    /* DivisionByZero         errors.hpp:18 */
    BCAD_CU_ERR_DOMAIN = 3,              /* DomainError            errors.hpp:24 */
    BCAD_CU_ERR_NON_DIFFERENTIABLE = 4,  /* NonDifferentiablePoint errors.hpp:29 */
    BCAD_CU_ERR_SHAPE_MISMATCH = 5,      /* ShapeMismatch          errors.hpp:33 */
    BCAD_CU_ERR_ARITY_MISMATCH = 6,      /* ArityMismatch          errors.hpp:37 */
    BCAD_CU_ERR_SEED_SHAPE_MISMATCH = 7, /* SeedShapeMismatch      errors.hpp:41 */
    BCAD_CU_ERR_UNKNOWN_PRIMITIVE = 8,   /* UnknownPrimitive       errors.hpp:45 */
    BCAD_CU_ERR_NON_FINITE = 9,          /* NonFiniteValue         errors.hpp:49 */
    BCAD_CU_ERR_SIZE_GUARD = 10,         /* SizeGuardExceeded      errors.hpp:53 */
    BCAD_CU_ERR_CONFIG = 11,             /* ConfigError            errors.hpp:57 */
    BCAD_CU_ERR_IO = 12,                 /* IoError                errors.hpp:61 */
    BCAD_CU_ERR_EQUIVALENCE = 13,        /* EquivalenceFailure     errors.hpp:65 */
    BCAD_CU_ERR_GENERIC = 15,            /* Error                  errors.hpp:8  */
    BCAD_CU_ERR_CUDA = 100,              /* CUDA runtime failure (incl. no device) */
    BCAD_CU_ERR_NCCL = 101               /* NCCL failure / NCCL unavailable */
} bcad_cu_status;

typedef enum bcad_cu_dtype { BCAD_CU_F32 = 0, BCAD_CU_F64 = 1 } bcad_cu_dtype;

/* Dense row-major extent. Axes align from the FIRST axis; shorter shapes are
 * padded with trailing 1s (shape.hpp:13-16). rank 0 = scalar. */
typedef struct bcad_cu_shape {
    int32_t rank;
    int32_t reserved;
    int64_t dims[BCAD_CU_MAX_RANK];
} bcad_cu_shape;

/* Opaque handle to a registered device kernel body (static lifetime). */
typedef const struct bcad_cu_kernel_entry* bcad_cu_kernel;

/* ---------------------------------------------------------------- info */
int bcad_cu_version(void);
/* Thread-local message of the last non-OK status on this thread. */
const char* bcad_cu_last_error(void);
int bcad_cu_kernel_count(void);
const char* bcad_cu_kernel_name(int index);
/* Looks a kernel up by BroadcastKernel::name(). n_in / m_out must match the
 * registered arity (ARITY_MISMATCH) — kernel.hpp:30-35 range checks apply;
 * unknown names give UNKNOWN_PRIMITIVE (there is no CPU fallback). */
int bcad_cu_kernel_lookup(const char* name, int n_in, int m_out, bcad_cu_kernel* out);
int bcad_cu_kernel_arity(bcad_cu_kernel k, int* n_in, int* m_out);
/* 1 if the kernel's dual rules can raise (log/div/sqrt/abs/pow). */
int bcad_cu_kernel_may_raise(bcad_cu_kernel k);
/* Registers a user device body (the entry the BCAD_DEVICE_KERNEL macro of
 * include/bcad/device_kernel.cuh builds in the user's nvcc translation unit:
 * forward and pullback launchers instantiated on the user's functor). The
 * entry must have static lifetime. A name that is already registered is
 * refused (CONFIG): a second body can never shadow or replace a first one.
 * Replaces the reference's type-erased body capture, kernel.hpp:26-43. */
int bcad_cu_register_kernel(const struct bcad_cu_kernel_entry* entry);

/* First-axis broadcast of n shapes (shape.hpp:70-90). */
int bcad_cu_broadcast_shape(int n, const bcad_cu_shape* shapes, bcad_cu_shape* out);

/* ------------------------------------------------------------ compute */
/* Fused forward: one visit per output cell evaluates the kernel body on
 * N-wide duals seeded x_j + e_j and writes
 *   primal_out[i]           (M pointers, entries may be NULL; array may be NULL)
 *   partials_out[i*N + j]   (M*N pointers at OUTPUT shape; entries may be NULL)
 * If partials_out == NULL the real-valued body runs instead (broadcast_apply).
 * Inputs are read in place through stride-0 broadcasting; nothing is
 * expanded. For kernels that may raise, the call synchronizes `stream` and
 * returns the status of the lowest failing cell, with the output index in
 * bcad_cu_last_error() ("... at output index (r, c)", forward.hpp:137-146). */
int bcad_cu_forward(bcad_cu_kernel k, int dtype, int n_in, const void* const* in,
                    const bcad_cu_shape* in_shapes, int m_out, void* const* primal_out,
                    void* const* partials_out, void* stream);

/* Bytes of device workspace bcad_cu_pullback needs for this problem: the
 * fp64 per-tile partials of reductions that span several CTAs, and the
 * completion tickets with which the last-arriving CTA of each strip combines
 * them inside the same launch. A workspace must be zero-filled once after
 * allocation (bcad_cu_pullback_workspace_init); every pullback leaves its
 * tickets zero again, so it can be reused by any later pullback without
 * re-initialisation. Concurrent pullbacks need separate workspaces. */
int bcad_cu_pullback_workspace(bcad_cu_kernel k, int dtype, int n_in, const bcad_cu_shape* in_shapes,
                               int m_out, size_t* bytes);
/* Zero-fills a freshly allocated workspace (stream-ordered memset). */
int bcad_cu_pullback_workspace_init(void* workspace, size_t bytes, void* stream);

/* Device kernel launches one bcad_cu_pullback of this problem issues with
 * aligned pointers, every input taking an adjoint and the workspace
 * bcad_cu_pullback_workspace sizes (tiled 2-D path: 1 = K2 alone, 2 = K2 +
 * K2f; generic rank-N path: 1-5). */
int bcad_cu_pullback_launches(bcad_cu_kernel k, int dtype, int n_in, const bcad_cu_shape* in_shapes, int m_out,
                              int* launches);

/* Pullback of one mixed node: for every input j with in_adj[j] != NULL,
 *   in_adj[j] (=|+=) sum over outputs i with out_adj[i] != NULL of
 *                    (out_adj[i] (.) D_ij) sum-reduced over the axes input j
 *                    was broadcast along,
 * where D_ij = partials[i*N + j] (CacheForward) or, when partials == NULL,
 * is recomputed from `in` in the same pass (RecomputeReverse). accumulate[j]
 * != 0 adds into the existing slot (tape.hpp:179-183), 0 overwrites it as a
 * freshly zeroed slot would be. Full-shape adjoints use the reference's
 * element arithmetic; reduced adjoints accumulate in fp64 in a fixed,
 * run-to-run deterministic order with no floating-point atomics.
 * in_adj pointers must not alias one another. */
int bcad_cu_pullback(bcad_cu_kernel k, int dtype, int n_in, const bcad_cu_shape* in_shapes, int m_out,
                     const void* const* out_adj, const void* const* partials, const void* const* in,
                     void* const* in_adj, const unsigned char* accumulate, void* workspace,
                     size_t workspace_bytes, void* stream);

/* acc (+)= contribution at acc's shape: sum-reduces over axes acc lacks or
 * expands along axes contribution lacks (broadcast.hpp:210-217). zero_first
 * != 0 treats acc as a freshly zero-initialised slot. */
int bcad_cu_scatter_add(int dtype, void* acc, const bcad_cu_shape* acc_shape, const void* contrib,
                        const bcad_cu_shape* contrib_shape, int zero_first, void* stream);

/* Transcendental evaluations (exp, log, sin, cos, tanh, sigmoid on reals or
 * duals) executed by the device kernels so far, summed over devices
 * (reference counters.hpp EvalCounters::transcendental_evals). The first call
 * arms the census: launches made before it are not counted; after it, every
 * body-evaluating launch is followed by a census launch that re-runs the body
 * per cell on counting scalars (the production kernels carry no counting
 * code). Synchronises every device that has counted. */
int bcad_cu_eval_counters(unsigned long long* transcendental_evals);
/* pause != 0: launches from this host thread stop counting until a matching
 * bcad_cu_count_pause(0) (nested). Used for the library's own probe launches
 * (the body check of BroadcastKernel), which the reference never runs. */
int bcad_cu_count_pause(int pause);

/* ptr[0..count) = value (dtype elements). */
int bcad_cu_fill(int dtype, void* ptr, int64_t count, double value, void* stream);

/* ------------------------------------------------------ device / memory */
int bcad_cu_device_count(int* count);
int bcad_cu_set_device(int device);
int bcad_cu_get_device(int* device);
/* Stream-ordered allocation from the device's caching pool (release
 * threshold unbounded, so steady-state steps do not touch the driver). */
int bcad_cu_malloc(void** ptr, size_t bytes, void* stream);
int bcad_cu_free(void* ptr, void* stream);
int bcad_cu_host_alloc(void** ptr, size_t bytes); /* pinned host memory */
int bcad_cu_host_free(void* ptr);
/* 1 if `ptr` is page-locked (pinned / registered) host memory, else 0. */
int bcad_cu_host_is_pinned(const void* ptr);
/* kind: 0 host->device, 1 device->host, 2 device->device */
int bcad_cu_memcpy(void* dst, const void* src, size_t bytes, int kind, void* stream);
int bcad_cu_memset(void* ptr, int value, size_t bytes, void* stream);
/* n independent copies of one kind (0 host->device, 1 device->host, 2
 * device->device) enqueued on `stream` with ONE call: host transfers through
 * cudaMemcpyBatchAsync (a per-copy loop on the legacy NULL stream), device
 * copies as one multi-buffer copy kernel. The copies must not overlap. */
int bcad_cu_memcpy_batch(size_t n, void* const* dsts, const void* const* srcs, const size_t* sizes, int kind,
                         void* stream);
int bcad_cu_stream_create(void** stream);
int bcad_cu_stream_destroy(void* stream);
int bcad_cu_stream_synchronize(void* stream);
int bcad_cu_device_synchronize(void);
/* Stream ordering between streams (fork/join of pipelined host steps):
 * timing-disabled events. */
int bcad_cu_event_create(void** event);
int bcad_cu_event_destroy(void* event);
int bcad_cu_event_record(void* event, void* stream);
int bcad_cu_stream_wait_event(void* stream, void* event);
/* CUDA graphs of enqueued work: capture everything enqueued on `stream` (and
 * on streams joined to it through events) between begin and end into an
 * executable graph; replay it with one launch. Capture is thread-local. */
int bcad_cu_graph_capture_begin(void* stream);
int bcad_cu_graph_capture_end(void* stream, void** graph_exec);
int bcad_cu_graph_launch(void* graph_exec, void* stream);
int bcad_cu_graph_destroy(void* graph_exec);

/* ------------------------------------------------------ multi-GPU (NCCL) */
/* NCCL is loaded at run time (dlopen libnccl.so.2); without it these return
 * BCAD_CU_ERR_NCCL. The unique id is 128 opaque bytes, exchanged by the
 * caller (e.g. over torch.distributed) before bcad_cu_comm_init. */
int bcad_cu_nccl_unique_id(unsigned char id[128]);
int bcad_cu_comm_init(void** comm, int nranks, const unsigned char id[128], int rank);
int bcad_cu_comm_destroy(void* comm);
/* Number of ranks in the communicator (ncclCommCount). */
int bcad_cu_comm_count(void* comm, int* nranks);
/* In-place sum over ranks of n_bufs device buffers (counts in elements), one
 * grouped NCCL launch on `stream`: the reduced adjoints of batch-broadcast
 * arguments after a batch-sharded pullback. */
int bcad_cu_allreduce_adjoints(void* const* bufs, const size_t* counts, int n_bufs, int dtype, void* comm,
                               void* stream);

/* ------------------------------------------ fused pullback allreduce
 * A peer-memory group for the compute+collective form of the sharded
 * pullback: K2's cross-CTA finisher (K2f) stores its fp64 column sums
 * straight into every rank's buffer over NVLink and, after a flag exchange,
 * each rank adds the world's sums in rank order — the allreduce of the
 * batch-broadcast ((1,H)-class) adjoints happens inside the pullback's own
 * last kernel, with no separate collective launch, identical bits on every
 * rank and one fp32 rounding of the fp64 world sum (the NCCL path rounds each
 * rank's partial). One group per rank (one process per GPU, or several ranks
 * in one process): create returns this rank's handle blob, every rank
 * gathers all blobs in rank order (e.g. torch.distributed all_gather) and
 * connects. max_elems bounds the reduced elements of one pullback
 * (n_col_args * H). Every rank must issue the same sequence of
 * bcad_cu_pullback_allreduce calls; a rank whose peers never arrive traps
 * after 30 s (no silent hang). Replaces bcad_cu_pullback +
 * bcad_cu_allreduce_adjoints for the sharded step. */
#define BCAD_CU_PEER_HANDLE_BYTES 128
typedef struct bcad_cu_peer_group_s* bcad_cu_peer_group;
int bcad_cu_peer_group_create(int rank, int world, size_t max_elems, bcad_cu_peer_group* out,
                              unsigned char handle[BCAD_CU_PEER_HANDLE_BYTES]);
int bcad_cu_peer_group_connect(bcad_cu_peer_group group, const unsigned char* handles);
int bcad_cu_peer_group_destroy(bcad_cu_peer_group group);
int bcad_cu_pullback_allreduce(bcad_cu_kernel k, int dtype, int n_in, const bcad_cu_shape* in_shapes, int m_out,
                               const void* const* out_adj, const void* const* partials, const void* const* in,
                               void* const* in_adj, const unsigned char* accumulate, void* workspace,
                               size_t workspace_bytes, bcad_cu_peer_group group, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BCAD_CU_H */
