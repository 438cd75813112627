/*
 * ltgp_refabi.h — engine binding for the reference-typed drop-in
 * (libltgp_refabi.so, paper_1902_09215_b200/host/evolve_cuda.cpp).
 *
 * libltgp_refabi.so defines, against the reference's UNMODIFIED headers
 * (/root/reference/proj/include/ltgp/evolve.hpp and eval.hpp), the
 * declarations a GPquick-style code base links against:
 *   ltgp::evaluate_population      evolve.hpp:108-109
 *   ltgp::execute_generation       evolve.hpp:111-117
 *   ltgp::evaluate_individual      evolve.hpp:106
 *   ltgp::eval_batch_raw           eval.hpp:73-74
 *   ltgp::eval_batch               eval.hpp:78-79
 *   ltgp::EvalStack::reserve_frames / grow   eval.hpp:27-52
 * on top of the C ABI in ltgp_cuda.h. ExecContext (evolve.hpp:95-100) has no
 * engine member, so the engine is found through the address of the context's
 * worker pool (ExecContext::pool, the caller's std::vector<WorkerState>):
 * bind one with ltgp_ref_bind_engine, or let the first call create a default
 * engine (devices 0.. one per RunConfig::worker_count, round robin over the
 * visible GPUs, node_limit = RunConfig::node_limit).
 *
 * Plain C: no exceptions or C++ types cross these entry points (0 = ok,
 * < 0 = error, message in ltgp_last_error()).
 */
#ifndef LTGP_REFABI_H
#define LTGP_REFABI_H

#include "ltgp_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Children genomes after execute_generation: copied back into
   Individual::genome (every child, one device-to-host copy each). Without the
   flag they stay on the device and Individual::genome is left empty; size,
   depth, fitness and hits are always filled, so a caller that plans from
   Individual::size needs no host genomes. */
#define LTGP_REF_MATERIALIZE_GENOMES 1

/* Bind engine e to the worker pool at pool_key (&ExecContext::pool). The
   caller keeps ownership of e. Replaces a previous binding of that key. */
int ltgp_ref_bind_engine(const void* pool_key, ltgp_engine* e, int flags);

/* Drop the binding of pool_key (destroys the engine if the binding created
   it). */
int ltgp_ref_unbind(const void* pool_key);

/* The engine bound to pool_key (NULL if none yet). */
ltgp_engine* ltgp_ref_engine(const void* pool_key);

#ifdef __cplusplus
}
#endif
#endif
