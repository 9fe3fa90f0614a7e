// layers.cpp -- one layer of the forward and of the backward of bns_epoch, per layer kind: GraphSAGE-mean / GCN
// aggregate-first (a6, a7, a9, a10), GraphSAGE transform-first (R42), GAT (f4, R45).  Each function only sequences
// kernel launches on the context stream; bns_epoch (api.cpp) does the exchanges, dropout, the loss and the reverse
// exchange around them.
#include "common.h"
#include "kernels.h"
#include "layers.h"

namespace bns {

namespace {
size_t tsz(const Ctx& c) { return c.prec == BNS_BF16 ? 2 : 4; }

// f4 / R45 GAT scalars of layer l (1-based): el, er over the stacked rows, softmax max / 1/Σ over inner rows, then
// one shared tail [c, selfds, del (inner) ; der, q / r (stacked)]
struct GatBufs {
    float *el, *er, *m, *inv, *cdot, *selfds, *del, *der, *qr;
};
GatBufs gat_bufs(const Ctx& c, int l) {
    const int64_t n_in = c.plan.n_in, R = n_in + c.halo_cap, L = c.L;
    GatBufs b;
    b.el = c.d_gat + (int64_t)(l - 1) * 2 * R;
    b.er = b.el + R;
    b.m = c.d_gat + 2 * L * R + (int64_t)(l - 1) * 2 * n_in;
    b.inv = b.m + n_in;
    b.cdot = c.d_gat + 2 * L * R + 2 * L * n_in;
    b.selfds = b.cdot + n_in;
    b.del = b.selfds + n_in;
    b.der = b.del + n_in;
    b.qr = b.der + R;
    return b;
}
}  // namespace

// f4 / R45 forward: Y = Hin W, el / er, softmax statistics, pre = Σ alpha Y (+ self), ReLU / fp32 logits
void forward_layer_gat(Ctx& c, const EpochView& v, int l, void* Hin) {
    const int L = c.L;
    const int64_t n_in = c.plan.n_in;
    const int64_t din = c.dp[l - 1], dout = c.dp[l];
    // f4 / R45: Y = Hin W on every stacked row (tcgen05), el / er, softmax statistics, then
    // pre_v = Σ_u alpha_vu Y_u + alpha_vv Y_v with ReLU (hidden) or fp32 logits (last) in the SpMM epilogue
    const bool last = (l == L);
    const int64_t rows = n_in + c.n_halo;
    const GatBufs GB = gat_bufs(c, l);
    float* el = GB.el;
    float* er = GB.er;
    float* gm = GB.m;
    float* ginv = GB.inv;
    const float* al = c.Wpad[l - 1] + din * dout;
    {
        PhaseTimer t(c, BNS_PH_GEMM_FWD);
        if (c.use_tc)
            gemm_fwd_tc(c, rows, dout, Hin, din, din, nullptr, 0, din, c.WT[l - 1], c.wkw[l - 1], c.d_tfy,
                        dout, false, false);
        else
            gemm_fwd(c, rows, dout, Hin, din, din, nullptr, 0, din, c.Wt[l - 1], dout, c.d_tfy, dout, false,
                     false);
    }
    PhaseTimer t(c, BNS_PH_SPMM_FWD);
    launch_gat_scores(c, c.d_tfy, dout, rows, (int32_t)dout, al, al + dout, el, er);
    launch_gat_stats(c, v.fsegs, c.n_seg_fwd, v.fcol, v.fsplit, c.n_split_fwd, el, er, gm, ginv);
    SpmmArgs a{};
    a.mode = GAT_FWD;
    a.segs = v.fsegs;
    a.n_segs = c.n_seg_fwd;
    a.col = v.fcol;
    a.src = c.d_tfy;
    a.ld_src = dout;
    a.self = c.d_tfy;
    a.ld_self = dout;
    a.out = last ? (void*)c.d_logits : c.H[l];
    a.ld_out = dout;
    a.d = (int32_t)dout;
    a.n_in = n_in;
    a.inv_p = 1.f;
    a.sc = 3;
    a.gat_el = el;
    a.gat_er = er;
    a.gat_m = gm;
    a.gat_inv = ginv;
    a.partial = c.d_partial;
    a.split = v.fsplit;
    a.n_split = c.n_split_fwd;
    a.relu = last ? 0 : 1;
    a.out_f32 = last ? 1 : 0;
    launch_spmm(c, a);
    return;
}

// R42 forward: [Y | S] = Hin [W_top | W_bot], pre = (1/deg) Σ c_u Y_u + S, ReLU / fp32 logits
void forward_layer_tf(Ctx& c, const EpochView& v, int l, void* Hin) {
    const int L = c.L;
    const int64_t n_in = c.plan.n_in;
    const size_t ts = tsz(c);
    const int64_t din = c.dp[l - 1], dout = c.dp[l];
    const float inv_p = v.inv_p;
    // R42 transform-first: [Y | S] = Hin [W_top | W_bot] on every stacked row, then
    // pre_v = (1/deg_G(v)) Σ_u c_u Y_u + S_v with ReLU (hidden) or fp32 logits (last) in the SpMM epilogue
    const bool last = (l == L);
    const int64_t rows = n_in + c.n_halo;
    {
        PhaseTimer t(c, BNS_PH_GEMM_FWD);
        if (c.use_tc)
            gemm_fwd_tc(c, rows, 2 * dout, Hin, din, din, nullptr, 0, din, c.WTtf[l - 1], (din + 63) / 64 * 64,
                        c.d_tfy, 2 * dout, false, false);
        else
            gemm_fwd(c, rows, 2 * dout, Hin, din, din, nullptr, 0, din, c.Wcat[l - 1], 2 * dout, c.d_tfy,
                     2 * dout, false, false);
    }
    PhaseTimer t(c, BNS_PH_SPMM_FWD);
    SpmmArgs a{};
    a.mode = SAGE_FWD_TF;
    a.segs = v.fsegs;
    a.hub_n = v.fhub_n;
    a.hub_base = v.fhub_base;
    a.n_segs = c.n_seg_fwd;
    a.col = v.fcol;
    a.src = c.d_tfy;
    a.ld_src = 2 * dout;
    a.self = static_cast<char*>(c.d_tfy) + dout * ts;
    a.ld_self = 2 * dout;
    a.out = last ? (void*)c.d_logits : c.H[l];
    a.ld_out = dout;
    a.d = (int32_t)dout;
    a.n_in = n_in;
    a.inv_p = inv_p;
    a.nscale = c.nscale;
    a.rowscale = c.d_deg_in;
    a.partial = c.d_partial;
    a.split = c.fwd_mode == 0 ? c.d_split_sf : (c.fwd_mode == 1 ? c.d_split_bwd : c.d_split_fwd);
    a.n_split = c.n_split_fwd;
    a.relu = last ? 0 : 1;
    a.out_f32 = last ? 1 : 0;
    launch_spmm(c, a);
    return;
}

// a6 + a7: Z = aggregation of Hin (SAGE mean / GCN P), pre = [Z | Hin] W (SAGE) or Z W (GCN), ReLU / logits
void forward_layer_std(Ctx& c, const EpochView& v, int l, void* Hin) {
    const int L = c.L;
    const int64_t n_in = c.plan.n_in;
    const bool sage = c.layer == BNS_LAYER_SAGE_MEAN;
    const int64_t din = c.dp[l - 1], dout = c.dp[l];
    const float inv_p = v.inv_p;
    {
        PhaseTimer t(c, BNS_PH_SPMM_FWD);
        SpmmArgs a{};
        a.mode = sage ? SAGE_FWD : GCN_FWD;
        a.segs = v.fsegs;
        a.hub_n = v.fhub_n;
        a.hub_base = v.fhub_base;
        a.n_segs = c.n_seg_fwd;
        a.col = v.fcol;
        a.src = Hin;
        a.ld_src = din;
        a.out = c.Z[l];
        a.ld_out = din;
        a.d = (int32_t)din;
        a.n_in = n_in;
        a.inv_p = inv_p;
        a.nscale = c.nscale;
        a.rowscale = sage ? c.d_deg_in : c.d_rs_in;
        a.cscale = c.d_cscale;
        a.partial = c.d_partial;
        a.split = c.fwd_mode == 0 ? c.d_split_sf : (c.fwd_mode == 1 ? c.d_split_bwd : c.d_split_fwd);
        a.n_split = c.n_split_fwd;
        launch_spmm(c, a);
    }
    {
        PhaseTimer t(c, BNS_PH_GEMM_FWD);
        const bool last = (l == L);
        void* out = last ? (void*)c.d_logits : c.H[l];
        if (c.use_tc)
            gemm_fwd_tc(c, n_in, dout, c.Z[l], din, din, sage ? Hin : nullptr, sage ? din : 0, din, c.WT[l - 1],
                        c.wkw[l - 1], out, dout, !last, last);
        else if (sage)
            gemm_fwd(c, n_in, dout, c.Z[l], din, din, Hin, din, din, c.Wt[l - 1], dout, out, dout, !last, last);
        else
            gemm_fwd(c, n_in, dout, c.Z[l], din, din, nullptr, 0, din, c.Wt[l - 1], dout, out, dout, !last, last);
    }
}

// f4 / R45 backward: dW, da_l, da_r into the gradient buffer, dX (l > 1) into c.d_dx
void backward_layer_gat(Ctx& c, const EpochView& v, int l, void* Hin) {
    const int L = c.L;
    const int64_t n_in = c.plan.n_in;
    const int64_t din = c.dp[l - 1], dout = c.dp[l];
    // f4 / R45 backward (g = dPre): c_v = g_v . pre_v, del_v / der_u = Σ ds over the forward / transposed
    // segments, dY by the weighted SpMM^T, dW = Hin^T dY, da_l = Σ del Y, da_r = Σ der Y, dX = dY W^T
    const bool last = (l == L);
    const int64_t rows = n_in + c.n_halo;
    const GatBufs GB = gat_bufs(c, l);
    float* el = GB.el;
    float* er = GB.er;
    float* gm = GB.m;
    float* ginv = GB.inv;
    float* cdot = GB.cdot;
    float* selfds = GB.selfds;
    float* del = GB.del;
    float* der = GB.der;
    float* qr = GB.qr;
    const float* al = c.Wpad[l - 1] + din * dout;
    float* g = c.d_gflat + c.goff[l - 1];
    {
        PhaseTimer t(c, BNS_PH_GEMM_BWD);   // Y again (same GEMM, same values)
        if (c.use_tc)
            gemm_fwd_tc(c, rows, dout, Hin, din, din, nullptr, 0, din, c.WT[l - 1], c.wkw[l - 1], c.d_tfy,
                        dout, false, false);
        else
            gemm_fwd(c, rows, dout, Hin, din, din, nullptr, 0, din, c.Wt[l - 1], dout, c.d_tfy, dout, false,
                     false);
    }
    {
        PhaseTimer t(c, BNS_PH_SPMM_BWD);
        launch_gat_rowdots(c, c.d_dpre, last ? (const void*)c.d_logits : c.H[l], last, c.d_tfy, dout,
                           (int32_t)dout, el, er, gm, ginv, cdot, selfds);
        // del_v = g_v . Q_v - c_v q_v + self, Q_v = Σ_u w_vu Y_u (w = alpha LeakyReLU')
        SpmmArgs aq{};
        aq.mode = GAT_RAW;
        aq.segs = v.fsegs;
        aq.n_segs = c.n_seg_fwd;
        aq.col = v.fcol;
        aq.src = c.d_tfy;
        aq.ld_src = dout;
        aq.out = c.d_gat_qp;
        aq.ld_out = dout;
        aq.d = (int32_t)dout;
        aq.n_in = n_in;
        aq.inv_p = 1.f;
        aq.sc = 5;
        aq.gat_el = el;
        aq.gat_er = er;
        aq.gat_m = gm;
        aq.gat_inv = ginv;
        aq.partial = c.d_partial;
        aq.split = v.fsplit;
        aq.n_split = c.n_split_fwd;
        launch_spmm(c, aq);
        launch_gat_wsum(c, 0, v.fsegs, c.n_seg_fwd, v.fcol, v.fsplit, c.n_split_fwd, el, er, gm, ginv, cdot, qr);
        launch_gat_final(c, 0, c.d_dpre, c.d_gat_qp, dout, (int32_t)dout, n_in, cdot, qr, selfds, del);
        // der_u = Y_u . P_u - r_u + self, P_u = Σ_v w_vu g_v over the transposed segments
        SpmmArgs ap = aq;
        ap.segs = v.bsegs;
        ap.n_segs = c.n_seg_bwd;
        ap.col = v.bcol;
        ap.src = c.d_dpre;
        ap.sc = 6;
        ap.split = v.bsplit;
        ap.n_split = c.n_split_bwd;
        launch_spmm(c, ap);
        launch_gat_wsum(c, 1, v.bsegs, c.n_seg_bwd, v.bcol, v.bsplit, c.n_split_bwd, el, er, gm, ginv, cdot, qr);
        launch_gat_final(c, 1, c.d_tfy, c.d_gat_qp, dout, (int32_t)dout, rows, cdot, qr, selfds, der);
        SpmmArgs a{};
        a.mode = GAT_BWD;
        a.segs = v.bsegs;
        a.n_segs = c.n_seg_bwd;
        a.col = v.bcol;
        a.src = c.d_dpre;
        a.ld_src = dout;
        a.out = c.d_gat_dy;
        a.ld_out = dout;
        a.d = (int32_t)dout;
        a.n_in = n_in;
        a.inv_p = 1.f;
        a.sc = 4;
        a.gat_el = el;
        a.gat_er = er;
        a.gat_m = gm;
        a.gat_inv = ginv;
        a.gat_al = al;
        a.gat_ar = al + dout;
        a.gat_del = del;
        a.gat_der = der;
        a.partial = c.d_partial;
        a.split = v.bsplit;
        a.n_split = c.n_split_bwd;
        launch_spmm(c, a);
    }
    {
        PhaseTimer t(c, BNS_PH_GEMM_BWD);
        auto wgrad = c.use_tc ? gemm_wgrad_tc : gemm_wgrad;
        auto dxg = c.use_tc ? gemm_dx_tc : gemm_dx;
        wgrad(c, rows, din, dout, Hin, din, c.d_gat_dy, dout, g, dout);
        launch_gat_da(c, c.d_tfy, dout, (int32_t)dout, del, n_in, g + din * dout);
        launch_gat_da(c, c.d_tfy, dout, (int32_t)dout, der, rows, g + (din + 1) * dout);
        if (l > 1) dxg(c, rows, din, dout, c.d_gat_dy, dout, c.Wt[l - 1], dout, c.d_dx, din, nullptr, 0);
    }
}

// R42 backward: dY by the narrow SpMM^T, dW_top / dW_bot, dX (l > 1) into c.d_dx
void backward_layer_tf(Ctx& c, const EpochView& v, int l, void* Hin) {
    const int64_t n_in = c.plan.n_in;
    const size_t ts = tsz(c);
    const int64_t din = c.dp[l - 1], dout = c.dp[l];
    const float inv_p = v.inv_p;
    // R42 transform-first backward: dY_u = c_u Σ_v dPre_v / deg_G(v) over every stacked row (SpMM^T at the
    // narrow width), dW_top = Hin^T dY, dW_bot = Hin_inner^T dPre, dX = [dY | dPre] [W_top | W_bot]^T
    const bool eb = c.sampler != BNS_SAMPLER_BNS;
    const int64_t rows = n_in + c.n_halo;
    {
        PhaseTimer t(c, BNS_PH_SPMM_BWD);
        SpmmArgs a{};
        a.mode = SAGE_BWD;
        a.segs = eb ? c.d_eseg_bwd : c.d_seg_bwd;
        a.n_segs = c.n_seg_bwd;
        a.col = eb ? c.d_ind_tcol : c.d_tcol;
        a.src = c.d_dxcat;       // dPre_v / deg_G(v), written by k_xent / k_relu_mask
        a.ld_src = dout;
        a.out = c.d_tfy;
        a.ld_out = 2 * dout;
        a.self = nullptr;
        a.d = (int32_t)dout;
        a.n_in = n_in;
        a.inv_p = inv_p;
        a.nscale = c.nscale;
        a.partial = c.d_partial;
        a.split = eb ? c.d_esplit_bwd : c.d_split_bwd;
        a.n_split = c.n_split_bwd;
        launch_spmm(c, a);
    }
    {
        PhaseTimer t(c, BNS_PH_GEMM_BWD);
        float* g = c.d_gflat + c.goff[l - 1];
        auto wgrad = c.use_tc ? gemm_wgrad_tc : gemm_wgrad;
        auto dxg = c.use_tc ? gemm_dx_tc : gemm_dx;
        // dPre: in the dPre half of d_tfy already (written there by the loss), else in d_dpre
        const bool in_tfy = tf_dpre_in_tfy(c, l);
        const void* dpre = in_tfy ? static_cast<const void*>(static_cast<char*>(c.d_tfy) + dout * ts) : c.d_dpre;
        const int64_t ldp = in_tfy ? 2 * dout : dout;
        if (c.use_tc) {   // dW_top (every stacked row) and dW_bot (inner rows) in one launch + one reduce
            gemm_wgrad2_tc(c, rows, n_in, din, dout, Hin, Hin, din, c.d_tfy, 2 * dout, dpre, ldp, g, dout);
        } else {
            wgrad(c, rows, din, dout, Hin, din, c.d_tfy, 2 * dout, g, dout);
            wgrad(c, n_in, din, dout, Hin, din, dpre, ldp, g + din * dout, dout);
        }
        if (l > 1) {   // dX = [dY | dPre] [W_top | W_bot]^T over every stacked row, one GEMM: halo rows have no dPre
            if (!in_tfy) {
                BNS_CUDA_HOLD(cudaMemcpy2DAsync(static_cast<char*>(c.d_tfy) + dout * ts, 2 * dout * ts, c.d_dpre,
                                           dout * ts, dout * ts, n_in, cudaMemcpyDeviceToDevice, c.stream));
                if (c.n_halo > 0)
                    BNS_CUDA_HOLD(cudaMemset2DAsync(static_cast<char*>(c.d_tfy) + (n_in * 2 + 1) * dout * ts, 2 * dout * ts,
                                               0, dout * ts, c.n_halo, c.stream));
            }
            dxg(c, rows, din, 2 * dout, c.d_tfy, 2 * dout, c.Wcat[l - 1], 2 * dout, c.d_dx, din, nullptr, 0);
        }
    }
}

// a9 + a10: dW, [dZ' | dXself] = dPre W^T, dX = transposed aggregation (l > 1) into c.d_dx
void backward_layer_std(Ctx& c, const EpochView& v, int l, void* Hin) {
    const int64_t n_in = c.plan.n_in;
    const size_t ts = tsz(c);
    const bool sage = c.layer == BNS_LAYER_SAGE_MEAN;
    const int64_t din = c.dp[l - 1], dout = c.dp[l];
    const float inv_p = v.inv_p;
    {
        PhaseTimer t(c, BNS_PH_GEMM_BWD);
        float* g = c.d_gflat + c.goff[l - 1];
        auto wgrad = c.use_tc ? gemm_wgrad_tc : gemm_wgrad;
        auto dxg = c.use_tc ? gemm_dx_tc : gemm_dx;
        if (sage && c.use_tc) {   // dW_z and dW_h share dPre: one launch, one split-K reduce
            gemm_wgrad2_tc(c, n_in, n_in, din, dout, c.Z[l], Hin, din, c.d_dpre, dout, c.d_dpre, dout, g, dout);
        } else {
            wgrad(c, n_in, din, dout, c.Z[l], din, c.d_dpre, dout, g, dout);
            if (sage) wgrad(c, n_in, din, dout, Hin, din, c.d_dpre, dout, g + din * dout, dout);
        }
        if (l > 1) {
            if (sage)
                dxg(c, n_in, 2 * din, dout, c.d_dpre, dout, c.Wt[l - 1], dout, c.d_dxcat, 2 * din, c.d_deg_in, din);
            else
                dxg(c, n_in, din, dout, c.d_dpre, dout, c.Wt[l - 1], dout, c.d_dxcat, din, c.d_rs_in, din);
        }
    }
    if (l == 1) return;   // R29: no gradient w.r.t. the input features
    {
        PhaseTimer t(c, BNS_PH_SPMM_BWD);
        SpmmArgs a{};
        const bool eb = c.sampler != BNS_SAMPLER_BNS;   // f3: the sampled transposed CSR of this epoch
        a.mode = sage ? SAGE_BWD : GCN_BWD;
        a.segs = eb ? c.d_eseg_bwd : c.d_seg_bwd;
        a.n_segs = c.n_seg_bwd;
        a.col = eb ? c.d_ind_tcol : c.d_tcol;
        a.src = c.d_dxcat;
        a.ld_src = sage ? 2 * din : din;
        a.out = c.d_dx;
        a.ld_out = din;
        a.self = static_cast<char*>(c.d_dxcat) + din * ts;
        a.ld_self = 2 * din;
        a.d = (int32_t)din;
        a.n_in = n_in;
        a.inv_p = inv_p;
        a.nscale = c.nscale;
        a.cscale = c.d_cscale;
        a.partial = c.d_partial;
        a.split = eb ? c.d_esplit_bwd : c.d_split_bwd;
        a.n_split = c.n_split_bwd;
        launch_spmm(c, a);
    }
}

}  // namespace bns
