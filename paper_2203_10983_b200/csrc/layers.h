// layers.h -- per-layer pieces of bns_epoch (layers.cpp) and the phase timer shared with api.cpp.
#pragma once
#include "common.h"

namespace bns {

// CUDA-event timing of one phase on the context stream (BNS_TIMING; read with BNS_Q_TIMES)
struct PhaseTimer {
    Ctx& c;
    int ph;
    size_t slot;
    PhaseTimer(Ctx& c_, int ph_) : c(c_), ph(ph_), slot(0) {
        if (!c.timing) return;
        slot = c.ev_used;
        if (slot + 2 > c.ev.size()) { ph = -1; return; }
        c.ev_used += 2;
        c.ev_phase[slot / 2] = ph;
        BNS_CUDA(cudaEventRecord(c.ev[slot], c.stream));
    }
    ~PhaseTimer() noexcept(false) {
        if (!c.timing || ph < 0) return;
        BNS_CUDA(cudaEventRecord(c.ev[slot + 1], c.stream));
    }
};


// the per-epoch structures every layer reads: forward segments / columns / split rows of this draw, the transposed
// ones, and the halo column scale c_u = 1/p (1 without halo)
struct EpochView {
    const Seg* fsegs; const int32_t* fcol; const int64_t* fsplit;
    int64_t fhub_n = 0, fhub_base = 0;   // forward list: hub segments first (SpmmArgs::hub_n)
    const Seg* bsegs; const int32_t* bcol; const int64_t* bsplit;
    float inv_p;
};

// R42 layer l = L with a dX (L > 1): the loss writes dPre into the dPre half of c.d_tfy (pitch 2 d_out, halo rows
// zeroed), the [dY | dPre] operand of the one dX GEMM -- no copy between the loss and the backward
inline bool tf_dpre_in_tfy(const Ctx& c, int l) {
    return l == c.L && l > 1 && c.layer == BNS_LAYER_SAGE_MEAN && ((c.tf_mask >> (l - 1)) & 1u);
}

// forward of layer l (1-based) from its (dropped-out) input Hin [inner ; halo]: H[l] (hidden) or the logits
void forward_layer_std(Ctx& c, const EpochView& v, int l, void* Hin);
void forward_layer_tf(Ctx& c, const EpochView& v, int l, void* Hin);
void forward_layer_gat(Ctx& c, const EpochView& v, int l, void* Hin);
// backward of layer l from c.d_dpre: the layer's weight gradient and, for l > 1, dX [inner ; halo] in c.d_dx
void backward_layer_std(Ctx& c, const EpochView& v, int l, void* Hin);
void backward_layer_tf(Ctx& c, const EpochView& v, int l, void* Hin);
void backward_layer_gat(Ctx& c, const EpochView& v, int l, void* Hin);

}  // namespace bns
