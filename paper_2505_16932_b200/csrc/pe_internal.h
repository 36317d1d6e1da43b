// Library-internal hooks between pe_api.cu (context, compute path) and
// pe_dist.cpp (NCCL communicator and the by-matrix sharded call).  Not part
// of the C ABI (include/pe.h); hidden C++ linkage.
#pragma once
#include <cuda_runtime.h>

#include "pe.h"

struct PeDist;                               // pe_dist.cpp: communicator, side stream, events

PeDist*& pe_ctx_dist(pe_ctx c);              // the context's distributed state (nullptr until attached)
int pe_ctx_device(pe_ctx c);
void pe_ctx_set_launches(pe_ctx c, int n);   // what pe_last_launch_count reports
void pe_set_error(const char* msg);          // pe_last_error_message of this thread
void pe_dist_free(PeDist* d);                // called by pe_destroy
// pe_polar_split's default all-reduce (user = the context): ncclAllReduce SUM
// over the context's communicator, on `stream`
extern "C" __attribute__((visibility("hidden"))) pe_status pe_comm_allreduce(void* buf, int64_t count, int dtype,
                                                                              void* user, void* stream);
