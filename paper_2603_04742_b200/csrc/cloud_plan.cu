// cloud_plan.cu -- see cloud_plan.hpp.
#include "cloud_plan.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <numeric>
#include <set>
#include <stdexcept>

#include "spmv/aggregate.hpp"

namespace cssc {

// Plan arrays are staged on the host and uploaded with ONE copy at the end
// of the constructor; put() hands out their future device addresses.
template <class T>
T* CloudPlan::put(const std::vector<T>& v) {
    const size_t off = (stage_.size() + 15) & ~size_t(15);
    const size_t bytes = sizeof(T) * v.size();
    if (off + bytes > arena_.bytes()) throw std::logic_error("plan arena too small");
    stage_.resize(off + bytes);
    if (bytes) std::memcpy(stage_.data() + off, v.data(), bytes);
    return reinterpret_cast<T*>(arena_.as<unsigned char>() + off);
}

CloudPlan::CloudPlan(GpuContext& ctx, const std::vector<uint64_t>& r,
                     const std::vector<uint64_t>& c, const std::vector<uint32_t>& slice,
                     int n_slices, const std::vector<const u64*>& a,
                     const std::vector<const u64*>& b, const std::vector<u64*>& out)
    : ctx_(ctx), n_((int)r.size()), ns_(n_slices) {
    const RnsParams& P = ctx.params();
    const int n = n_;
    if ((int)c.size() != n || (int)slice.size() != n || (int)a.size() != n || (int)b.size() != n ||
        (int)out.size() != ns_)
        throw std::invalid_argument("plan: inconsistent sizes");
    const size_t ctw = ctx.ct_words();
    const int L = P.cfg.L, LK = L + P.cfg.K, M = L + P.nB;

    std::vector<std::vector<spmv::RotStep>> steps(n);
    for (int i = 0; i < n; ++i) {
        if (r[i] * c[i] > (uint64_t)P.S) throw std::length_error("plan: chunk exceeds slot count");
        if (slice[i] >= (uint32_t)ns_) throw std::invalid_argument("plan: slice id out of range");
        steps[i] = spmv::rotation_schedule(r[i], c[i]);
    }
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int x, int y) { return steps[x].size() > steps[y].size(); });
    const int depth = n ? (int)steps[order[0]].size() : 0;
    // upper bound of all plan arrays (8-byte entries) plus 16-byte alignment slack
    arena_ = DevBuf(&ctx.pool(), 8 * ((size_t)(8 + 5 * depth) * std::max(n, 1) + 2 * (size_t)ns_ + 8) +
                                     16 * (size_t)(5 * depth + 16));

    prod_ = DevBuf(&ctx.pool(), sizeof(u64) * ctw * std::max(n, 1));
    if (depth >= 1) acc0_ = DevBuf(&ctx.pool(), sizeof(u64) * ctw * n);
    if (depth >= 2) acc1_ = DevBuf(&ctx.pool(), sizeof(u64) * ctw * n);
    T_ = DevBuf(&ctx.pool(), sizeof(u64) * std::max<size_t>(1, n) * ctx.mul_T_words());
    Z_ = DevBuf(&ctx.pool(), sizeof(u64) * std::max<size_t>(1, n) * ctx.mul_Z_words());
    D2_ = DevBuf(&ctx.pool(), sizeof(u64) * std::max<size_t>(1, n) * ctx.poly_words());
    DX_ = DevBuf(&ctx.pool(), sizeof(u64) * std::max<size_t>(1, n) * ctx.dx_words());
    ACC_ = DevBuf(&ctx.pool(), sizeof(u64) * std::max<size_t>(1, n) * ctx.ksacc_words());
    MT_ = DevBuf(&ctx.pool(), sizeof(u64) * std::max<size_t>(1, n) * ctw);

    auto prod_at = [&](int k) { return prod_.words() + (size_t)k * ctw; };
    auto acc_at = [&](int which, int k) {
        return (which == 0 ? acc0_.words() : acc1_.words()) + (size_t)k * ctw;
    };
    auto acc_after = [&](int k, int done) -> u64* {  // accumulator after `done` steps
        if (done == 0) return prod_at(k);
        return acc_at((done - 1) % 2, k);
    };

    std::vector<const u64*> va(n), vb(n), rlk(n, ctx.relin_key());
    std::vector<u64*> vp(n);
    for (int k = 0; k < n; ++k) {
        va[k] = a[order[k]];
        vb[k] = b[order[k]];
        vp[k] = prod_at(k);
    }
    A_ = put(va);
    B_ = put(vb);
    PROD_ = put(vp);
    RLK_ = put(rlk);

    const u64 C = sizeof(u64) * ctw, KEY = sizeof(u64) * ctx.ksk_words(),
              PT = sizeof(u64) * ctx.poly_words();
    stats_.chunks = n;
    stats_.slices = ns_;
    stats_.levels = depth;
    stats_.hbm_bytes = n ? (u64)n * 3 * C + KEY : 0;
    stats_.key_bytes = n ? KEY : 0;
    const bool fused = ctx.fused_key_switch();
    stats_.kernels = n ? (fused ? 11 : 14) : 0;  // each NTT is two kernels (column, block phase)
    stats_.limb_ntts = (u64)n * (7 * M + P.dnum * LK + 2 * LK);

    std::set<u32> all_keys;
    for (int l = 0; l < depth; ++l) {
        int items = 0;
        while (items < n && (int)steps[order[items]].size() > l) ++items;
        std::vector<const u64*> src(items), base(items), key(items);
        std::vector<u64*> o(items);
        std::vector<u32> gi(items);
        std::set<u32> lvl_keys;
        for (int k = 0; k < items; ++k) {
            const spmv::RotStep& s = steps[order[k]][l];
            u64* cur = acc_after(k, l);
            base[k] = cur;
            src[k] = s.from_accumulator ? cur : prod_at(k);
            o[k] = acc_at(l % 2, k);
            const u32 g = galois_element((int64_t)s.offset, P.n);
            key[k] = ctx.galois_key(g);
            // inverse Galois element in (Z/2N)^*: g^(N-1)
            u64 inv = 1, bb = g;
            const u64 two_n = 2 * (u64)P.n;
            for (u64 e = (u64)P.n - 1; e; e >>= 1) {
                if (e & 1) inv = inv * bb % two_n;
                bb = bb * bb % two_n;
            }
            gi[k] = (u32)inv;
            lvl_keys.insert(g);
            all_keys.insert(g);
        }
        Level lv;
        lv.items = items;
        lv.src = put(src);
        lv.base = put(base);
        lv.out = put(o);
        lv.key = put(key);
        lv.ginv = put(gi);
        levels_.push_back(lv);
        stats_.rotations += items;
        stats_.hbm_bytes += (u64)items * 3 * C + lvl_keys.size() * KEY;
        stats_.key_bytes += lvl_keys.size() * KEY;
        stats_.kernels += fused ? 4 : 7;
        stats_.limb_ntts += (u64)items * (P.dnum * LK + 2 * LK);
    }
    stats_.distinct_keys = all_keys.size();

    // masked inter-chunk accumulation
    std::map<uint64_t, int> mask_id;
    std::vector<int> ones;
    std::vector<int> item_mask(n);
    std::vector<const u64*> fin(n);
    for (int k = 0; k < n; ++k) {
        const uint64_t rr = r[order[k]];
        auto it = mask_id.find(rr);
        if (it == mask_id.end()) {
            it = mask_id.emplace(rr, (int)ones.size()).first;
            ones.push_back((int)rr);
        }
        item_mask[k] = it->second;
        fin[k] = acc_after(k, (int)steps[order[k]].size());
    }
    n_masks_ = (int)ones.size();
    MASKS_ = DevBuf(&ctx.pool(), sizeof(u64) * std::max<size_t>(1, n_masks_) * ctx.poly_words());
    ctx.encode_masks(ones, MASKS_.words());
    std::vector<int> off(ns_ + 1, 0), items_by_slice;
    std::vector<std::vector<int>> per(ns_);
    for (int k = 0; k < n; ++k) per[slice[order[k]]].push_back(k);
    for (int s = 0; s < ns_; ++s) {
        off[s + 1] = off[s] + (int)per[s].size();
        if (per[s].empty()) throw std::invalid_argument("plan: slice without chunks");
        items_by_slice.insert(items_by_slice.end(), per[s].begin(), per[s].end());
    }
    FINAL_ = put(fin);
    OUT_ = put(out);
    slice_off_ = put(off);
    slice_items_ = put(items_by_slice);
    item_mask_ = put(item_mask);
    stats_.hbm_bytes += (u64)n * 2 * C + (u64)n_masks_ * PT;
    stats_.kernels += n ? 5 : 0;
    stats_.limb_ntts += (u64)n * 2 * L + (u64)ns_ * 2 * L;
    if (!stage_.empty())
        cuda_check(cudaMemcpyAsync(arena_.as<void>(), stage_.data(), stage_.size(), cudaMemcpyHostToDevice,
                                   ctx.stream()),
                   "plan upload");
    ctx.synchronize();
}

CloudPlan::~CloudPlan() {
    if (exec_) cudaGraphExecDestroy(exec_);
    if (graph_) cudaGraphDestroy(graph_);
}

void CloudPlan::record() {
    if (n_ == 0) return;
    const RnsParams& P = ctx_.params();
    const int L = P.cfg.L, logn = P.cfg.logn;
    cudaStream_t st = ctx_.stream();
    ctx_.mul_relin_dev(A_, B_, PROD_, n_, T_.words(), Z_.words(), D2_.words(), DX_.words(),
                       ACC_.words(), RLK_);
    for (const Level& lv : levels_)
        ctx_.rotate_dev(lv.src, lv.ginv, lv.key, lv.base, lv.out, lv.items, DX_.words(),
                        ACC_.words());
    std::vector<int> qidx(L);
    std::iota(qidx.begin(), qidx.end(), 0);
    NttJob fwd = ctx_.job(nullptr, MT_.words(), 2 * L, qidx);
    fwd.src_items = FINAL_;
    launch_ntt(ctx_.dconsts(), logn, false, fwd, n_, st);
    u64* RES = T_.words();  // ns <= n results fit the multiply workspace
    launch_mask_accum(ctx_.dconsts(), P, MT_.words(), slice_off_, slice_items_, item_mask_,
                      MASKS_.words(), RES, ns_, st);
    NttJob inv = ctx_.job(RES, nullptr, 2 * L, qidx);
    inv.dst_items = OUT_;
    launch_ntt(ctx_.dconsts(), logn, true, inv, ns_, st);
}

void CloudPlan::run() {
    if (exec_) {
        cuda_check(cudaGraphLaunch(exec_, ctx_.stream()), "graph launch");
    } else {
        record();
    }
}

void CloudPlan::capture() {
    if (exec_ || n_ == 0) return;
    cudaStream_t st = ctx_.stream();
    cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
        record();
    } catch (...) {
        cudaGraph_t g;
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    cuda_check(cudaStreamEndCapture(st, &graph_), "end capture");
    cuda_check(cudaGraphInstantiate(&exec_, graph_, 0), "graph instantiate");
}

}  // namespace cssc
