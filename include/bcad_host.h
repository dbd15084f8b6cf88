/*
 * bcad_host.h — C-ABI of the end-to-end host call (libbcad_host.so), built on
 * the C++ drop-in API (include/bcad/*.hpp). One call is one reference step as
 * proj/src/bench.cpp:112-128 (run_cell_once) performs it — tape inputs from
 * HOST buffers, mixed_broadcast(kernel, ..., policy), backward(seeds), leaf
 * gradients back to HOST buffers — with every device step on `stream`.
 * This is the binding a non-C++ caller of the reference's
 * mixed_broadcast + Tape::backward (proj/include/bcad/mixed.hpp:49-99,
 * tape.hpp:185-211) would use.
 */
#ifndef BCAD_HOST_H
#define BCAD_HOST_H

#include <stdint.h>

#include "bcad_cu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* policy: 0 CacheForward, 1 RecomputeReverse (mixed.hpp:17-20).
 * host_seeds: m_out pointers at the output shape (entries may be NULL = no
 * adjoint for that output). host_grads: n_in pointers at the input shapes
 * (entries may be NULL = not wanted). Pinned host memory makes the copies
 * asynchronous. Returns a bcad_cu_status; the message is in
 * bcad_host_last_error(). */
int bcad_host_mixed_step(const char* kernel, int dtype, int n_in, const void* const* host_in,
                         const bcad_cu_shape* in_shapes, int m_out, int policy, const void* const* host_seeds,
                         void* const* host_primal, void* const* host_grads, int64_t* peak_cached_bytes,
                         void* stream);

/* The same step, enqueued without waiting for it (a serving / training loop
 * overlapping consecutive steps: the next step's uploads run during this
 * one's downloads). Requires the pipelined, prepared path: pinned host
 * buffers, a non-default stream, a problem large enough to chunk. Steps on
 * the SAME host buffers are ordered among themselves (a buffer is
 * overwritten only after the previous step has finished with it); give
 * consecutive steps different host gradient / primal buffers to let them
 * overlap. Results are on the host after bcad_host_synchronize(stream). */
int bcad_host_mixed_step_async(const char* kernel, int dtype, int n_in, const void* const* host_in,
                               const bcad_cu_shape* in_shapes, int m_out, int policy, const void* const* host_seeds,
                               void* const* host_primal, void* const* host_grads, void* stream);
/* Waits for every step this thread enqueued with bcad_host_mixed_step_async
 * (and for `stream`). */
int bcad_host_synchronize(void* stream);

/* cell_gradients (proj/include/bcad/hmlstm.hpp:123-142) on an n x n cell:
 * impl 0 mixed-cache, 1 mixed-recompute, 2 reverse-unfused (the 8-primitive
 * vectorised-select baseline, hmlstm.hpp:82-99). Inputs c, f, i, g (n*n),
 * z1, z2 (n) and the seed (n*n) are DEVICE pointers; they are copied into the
 * tape as the reference's Tape::input copies (tape.hpp:75-82). Gradients
 * dc, df, di, dg (n*n each) are written to DEVICE pointers. Reports the tape
 * size and peak_cached_bytes. Asynchronous on `stream` (no host sync). */
int bcad_host_cell_gradients(int impl, int dtype, int64_t n, const void* const* dev_in, const void* dev_seed,
                             void* const* dev_grads, int64_t* tape_nodes, int64_t* peak_cached_bytes, void* stream);

/* Row-chunk pipelining of bcad_host_mixed_step (a host-side schedule; the
 * math per row is unchanged): the batch axis (axis 0) is cut into chunks run
 * over four lane streams, so the host->device copy of one chunk, the kernels
 * of the next and the device->host copy of the previous overlap. Rows are
 * independent under first-axis broadcasting (shape.hpp:13-16); gradients of
 * batch-broadcast arguments (axis 0 of length 1, or scalars) are summed over
 * chunks in chunk order on the device. max_chunks: 0 = automatic (about 9 MiB
 * of host<->device traffic per chunk, at most 16 chunks), 1 = off (one tape
 * over the whole batch), k > 1 = at most k chunks. Kernels that may raise
 * always run one-shot so error indices match the reference. Process-wide. */
int bcad_host_set_pipeline(int max_chunks);

/* Prepared pipelined steps (default on): a pipelined call on pinned host
 * buffers keeps its device buffers, chunk plan and workspaces (a few entries
 * per thread, each at most 2 GiB of device memory) for later calls with the
 * same buffers, shapes and stream, which then only enqueue copies and
 * kernels. 0 disables and frees the calling thread's prepared steps. */
int bcad_host_set_prepared(int enable);

/* Deterministic inputs bit-identical to the reference's (proj/include/bcad/
 * rng.hpp:11-31, tensor.hpp:71-84): one Rng(seed) (mt19937_64) draws the n
 * tensors in order, volumes[j] elements each, kinds[j] 0 = random_pm1
 * (U(-1,1) from a 53-bit double), 1 = random_binary (exact {0,1}, p = 1/2).
 * Only elements [begin[j], begin[j] + count[j]) of tensor j are written to
 * host_out[j] (row blocks of a batch shard); the draws before them are
 * skipped. Host memory, one thread per tensor. */
int bcad_host_random_inputs(uint64_t seed, int dtype, int n, const int64_t* volumes, const int* kinds,
                            const int64_t* begin, const int64_t* count, void* const* host_out);

/* mix_seed(seed, salt) of proj/src/bench.cpp:31-37. */
uint64_t bcad_host_mix_seed(uint64_t seed, uint64_t salt);

const char* bcad_host_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* BCAD_HOST_H */
