// transport.h -- exchange / all-reduce interface used by bns_epoch (implemented in comm.cpp).
#pragma once
#include "common.h"

namespace bns {

struct Transport {
    virtual ~Transport() {}
    // Row-block all-to-allv: the rows this rank sends to peer j are src[src_off[j] .. src_off[j+1]); the rows it
    // receives from peer j land at dst[dst_off[j] .. dst_off[j+1]).  Offsets in rows (host arrays of m+1).
    virtual void exchange(Ctx& c, const void* src, const int64_t* src_off, void* dst, const int64_t* dst_off,
                          size_t rowbytes) = 0;
    // In-place sum over ranks of n fp32 and ns fp64 values.
    virtual void allreduce(Ctx& c, float* buf, int64_t n, double* scal, int64_t ns) = 0;
    // Setup-time sum of one host integer (blocking).
    virtual int64_t allreduce_host_i64(Ctx& c, int64_t v) = 0;
    // Raise a pending asynchronous communicator error.
    virtual void poll(Ctx& c) = 0;
};

Transport* make_transport(Ctx& c);

}  // namespace bns
