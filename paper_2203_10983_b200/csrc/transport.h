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
    // f1 peer-memory transports only (peer() == true): bns_epoch then calls begin_epoch once, halo_pull instead of
    // pack + exchange (forward layer l: the halo rows of H^(l-1) read from the owners), dx_buffer(l) as the layer-l
    // input-gradient buffer (alternating, so a peer may still read layer l+1's halo gradients), and grad_scatter
    // instead of reverse exchange + scatter-add (c.d_dx inner rows += the peers' halo gradients of this rank's rows).
    // allreduce() then leaves the sum in a second buffer and repoints c.d_gflat / c.d_scal at it.
    virtual bool peer() const { return false; }
    virtual void begin_epoch(Ctx&) {}
    virtual void halo_pull(Ctx&, int /*l*/, void* /*dst_halo*/, int64_t /*din*/) {}
    virtual void* dx_buffer(Ctx& c, int /*l*/);
    virtual void grad_scatter(Ctx&, int /*l*/, int64_t /*din*/) {}
    // the barrier of grad_scatter alone, the pull folded into the next ReLU-mask kernel: the peers' layer-l dX
    // pointer table and row deltas (false: not a peer transport)
    virtual bool grad_barrier(Ctx&, int /*l*/, const void* const** /*peer*/, const int64_t** /*delta*/) { return false; }
    // bns_destroy, before the context frees anything: make sure no peer still reads this rank's shared buffers
    // (peer transports skip the second barrier of the all-reduce, so a slower peer may be in k_sum_ptrs).
    virtual void shutdown(Ctx&) {}
};

inline void* Transport::dx_buffer(Ctx& c, int) { return c.d_dx; }

Transport* make_transport(Ctx& c);

}  // namespace bns
