// arc_loopback.h — the in-process loopback communicator (arc_loopback.cu), as
// the step's exchange code in arc_api.cu calls it.  Not part of the public ABI
// (the public entry points are arc_topk_loopback_* in include/arc_topk.h).
#pragma once
#include <cstddef>
#include <cuda_runtime.h>

#include "arc_topk.h"

namespace arc {

struct LoopbackComm;   // one emulated rank of a loopback group

int loopback_nranks(const LoopbackComm* c);
int loopback_rank(const LoopbackComm* c);
// all-gather: rank k's `bytes` land at recv + k * bytes on every rank
arc_status loopback_all_gather(LoopbackComm* c, const void* send, void* recv, size_t bytes, cudaStream_t s);
// all-reduce(sum) of `count` floats (in place allowed)
arc_status loopback_all_reduce_f32(LoopbackComm* c, const float* send, float* recv, size_t count, cudaStream_t s);
// all-reduce(sum) of `count` bfloat16 entries (the R25 wire): binary32 sum rounded once
arc_status loopback_all_reduce_bf16(LoopbackComm* c, const void* send, void* recv, size_t count, cudaStream_t s);
// all-to-all: scount[k] floats from send + sdispl[k] go to rank k; rcount[k]
// floats from rank k land at recv + rdispl[k]  (host arrays of G entries)
arc_status loopback_all_to_all_f32(LoopbackComm* c, const float* send, const size_t* scount, const size_t* sdispl,
                                   float* recv, const size_t* rcount, const size_t* rdispl, cudaStream_t s);

}  // namespace arc
