// cloud_plan.cu -- see cloud_plan.hpp.
//
// Level structure of the rotate-and-add trees.  rotation_schedule(r, c)
// (aggregate.cpp:19-34) interleaves "doubling" steps D_k (rotate the running
// accumulator) with "odd" steps O_k (rotate the ORIGINAL product, then add).
// An odd step's rotation does not depend on the accumulator, so the plan
// hoists every O_k into level 0, next to D_1, which also rotates the product.
// Its result RP_k is added where the reference adds it: right after D_k.
//   * k >= 2: the add is fused into the ModDown of the level computing D_k,
//     as an extra addend;
//   * k == 1: one elementwise add after level 0.
// The tree depth drops from numBits + popcount - 2 launches to numBits - 1.
// The ciphertexts are identical, because every rotation and addition is an
// exact function of its inputs, and the op ledger is unchanged.
#include "cloud_plan.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <set>
#include <stdexcept>

#include "nvtx_range.hpp"
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

namespace {

u32 inverse_galois(u32 g, int n) {
    const u64 two_n = 2 * (u64)n;
    u64 inv = 1, b = g;
    for (u64 e = (u64)n - 1; e; e >>= 1) {  // g^(N-1) = g^-1 in (Z/2N)^*
        if (e & 1) inv = inv * b % two_n;
        b = b * b % two_n;
    }
    return (u32)inv;
}

struct Tree {
    std::vector<u64> dbl;                  // doubling offsets D_1..D_m
    std::vector<std::pair<int, u64>> odd;  // (k, offset): O_k follows D_k
};

// One key-switch stage of a chunk's fold (fold mode, DESIGN 2.9): one doubling
// step D (offset d1) or two merged ones (d1, d2: acc + R(acc, d1) + R(acc, d2) +
// R(acc, d1 + d2)), plus the rotations of the product p its odd steps add
// (poff: O_a, O_a + d2 when merged, O_{a+1}); one ModDown per stage.
struct Stage {
    bool merged = false;
    u64 d1 = 0, d2 = 0;
    std::vector<u64> poff;
};

// Stage 0 is D_1 (+ O_1); after it, consecutive doubling steps pair greedily
// when no combined offset is 0 mod S (the oracle's plan fold, fold_relin = 2)
std::vector<Stage> make_stages(const Tree& t, u64 S, bool merge) {
    const int m = (int)t.dbl.size();
    std::vector<std::vector<u64>> odd_of(m + 1);
    for (const auto& [after, off] : t.odd) odd_of[after].push_back(off);
    std::vector<Stage> st;
    int a = 1;  // next doubling step D_a (1-based)
    while (a <= m) {
        Stage g;
        g.d1 = t.dbl[a - 1];
        const bool o1 = !odd_of[a].empty();
        if (merge && a >= 2 && a + 1 <= m) {
            const u64 d2 = t.dbl[a];
            const u64 o = o1 ? odd_of[a][0] : 0;
            if ((g.d1 + d2) % S != 0 && (!o1 || (o + d2) % S != 0)) {
                g.merged = true;
                g.d2 = d2;
                if (o1) {
                    g.poff.push_back(o);
                    g.poff.push_back(o + d2);
                }
                for (u64 x : odd_of[a + 1]) g.poff.push_back(x);
                st.push_back(g);
                a += 2;
                continue;
            }
        }
        for (u64 x : odd_of[a]) g.poff.push_back(x);
        st.push_back(g);
        a += 1;
    }
    return st;
}

Tree split_schedule(const std::vector<spmv::RotStep>& steps) {
    Tree t;
    for (const spmv::RotStep& s : steps) {
        if (s.from_accumulator)
            t.dbl.push_back(s.offset);
        else
            t.odd.emplace_back((int)t.dbl.size(), s.offset);
    }
    return t;
}

}  // namespace

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
    const int L = P.cfg.L, LK = L + P.cfg.K, M = P.mul_limbs();

    rows_.assign(ns_, 0);
    for (int i = 0; i < n; ++i)
        if (slice[i] < (uint32_t)ns_) rows_[slice[i]] = std::max<int>(rows_[slice[i]], (int)r[i]);
    out_off_.assign(ns_, 0);
    {
        size_t o = 0;
        for (int s2 = 0; s2 < ns_; ++s2) {
            out_off_[s2] = o;
            o += (size_t)rows_[s2];
        }
        maxdev_off_ = (4 * o + 15) & ~size_t(15);
    }
    std::vector<Tree> trees(n);
    size_t n_rot = 0, n_odd = 0;
    for (int i = 0; i < n; ++i) {
        if (r[i] * c[i] > (uint64_t)P.S) throw std::length_error("plan: chunk exceeds slot count");
        if (slice[i] >= (uint32_t)ns_) throw std::invalid_argument("plan: slice id out of range");
        const auto steps = spmv::rotation_schedule(r[i], c[i]);
        trees[i] = split_schedule(steps);
        n_rot += steps.size();
        n_odd += trees[i].odd.size();
    }
    // Folded level 0 (fused fixed-shape key switch, hoisting on): the products
    // of rotated chunks stay unrelinearised; level 0 hoists the ModUp + NTT of
    // their z1 and z2 and sums, per doubling item, the relinearisation of z2
    // and the rotations of z1 (key for phi_g(s)) and z2 (key for phi_g(s)^2)
    // into one ModDown; later levels are key-switch stages of one or two
    // doubling steps (DESIGN 2.9; the oracle restates it: plan fold, fold_relin
    // = 2, or 1 with CSSC_NO_MERGE=1)
    int ndbl = 0;
    for (int i = 0; i < n; ++i) ndbl += trees[i].dbl.empty() ? 0 : 1;
    const bool fold = ctx.fused_key_switch() && fixed_rns_shape(P) && std::getenv("CSSC_NO_KSY") == nullptr &&
                      std::getenv("CSSC_KS_CLUSTER") == nullptr && std::getenv("CSSC_NO_HOIST") == nullptr &&
                      ndbl > 0;
    const bool merge = fold && std::getenv("CSSC_NO_MERGE") == nullptr;
    std::vector<std::vector<Stage>> stages(n);
    size_t n_stage = 0;
    if (fold)
        for (int i = 0; i < n; ++i) {
            stages[i] = make_stages(trees[i], (u64)P.S, merge);
            n_stage += stages[i].size();
        }
    auto levels_of = [&](int i) { return fold ? stages[i].size() : trees[i].dbl.size(); };
    // chunks with more levels first: level l is a prefix of the items
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return levels_of(x) > levels_of(y); });
    const int depth = n ? (int)levels_of(order[0]) : 0;
    int nd = 0;  // chunks with at least one doubling step: items 0 .. nd-1
    while (nd < n && !trees[order[nd]].dbl.empty()) ++nd;
    fold_ = fold;
    nd_ = nd;
    stats_.relin_folded = fold ? (merge ? 2 : 1) : 0;

    arena_ = DevBuf(&ctx.pool(), 8 * ((size_t)(16 + 10 * std::max(depth, 1)) * std::max(n, 1) + 16 * n_odd +
                                      2 * (size_t)ns_ + 16) +
                                     16 * (size_t)(24 * depth + 40) + 8 * (6 * (size_t)n + 6 * n_odd) +
                                     8 * 48 * ((size_t)n * std::max(depth, 1) + 2 * n_stage));
    prod_ = DevBuf(&ctx.pool(), sizeof(u64) * ctw * std::max(n, 1));
    if (depth >= 1) acc0_ = DevBuf(&ctx.pool(), sizeof(u64) * ctw * n);
    if (depth >= 2) acc1_ = DevBuf(&ctx.pool(), sizeof(u64) * ctw * n);
    if (n_odd || n_stage) rp_ = DevBuf(&ctx.pool(), sizeof(u64) * ctw * std::max(n_odd, n_stage));
    T_ = DevBuf(&ctx.pool(), sizeof(u64) * std::max<size_t>(1, n) * ctx.mul_T_words());
    Z_ = DevBuf(&ctx.pool(), sizeof(u64) * std::max<size_t>(1, n) * ctx.mul_Z_words());
    D2_ = DevBuf(&ctx.pool(), sizeof(u64) * std::max<size_t>(1, n) * ctx.poly_words());
    const size_t ks_items = std::max<size_t>(1, (size_t)n + std::max(n_odd, n_stage));
    DX_ = DevBuf(&ctx.pool(), sizeof(u64) * std::max(ks_items, fold ? 2 * (size_t)nd : 1) * ctx.dx_words());
    ACC_ = DevBuf(&ctx.pool(), sizeof(u64) * ks_items * ctx.ksacc_words());
    MT_ = DevBuf(&ctx.pool(), sizeof(u64) * std::max<size_t>(1, n) * ctw);
    // hoisted ModUp factors (KsY) of every ciphertext a key switch reads: the
    // products, both accumulator arrays and the relinearisation's c2
    const bool hoist = ctx.fused_key_switch() && fixed_rns_shape(P) && std::getenv("CSSC_NO_KSY") == nullptr;
    const size_t pw = ctx.poly_words();
    if (hoist) {
        prodY_ = DevBuf(&ctx.pool(), sizeof(u64) * pw * std::max(n, 1));
        if (depth >= 1) accY0_ = DevBuf(&ctx.pool(), sizeof(u64) * pw * n);
        if (depth >= 2) accY1_ = DevBuf(&ctx.pool(), sizeof(u64) * pw * n);
        D2Y_ = DevBuf(&ctx.pool(), sizeof(u64) * pw * std::max(n, 1));
    }
    auto prodY_at = [&](int k) -> u64* { return hoist ? prodY_.words() + (size_t)k * pw : nullptr; };
    auto accY_at = [&](int which, int k) -> u64* {
        return hoist ? (which == 0 ? accY0_.words() : accY1_.words()) + (size_t)k * pw : nullptr;
    };
    auto yafter = [&](int k, int done) -> u64* { return done == 0 ? prodY_at(k) : accY_at((done - 1) % 2, k); };

    auto prod_at = [&](int k) { return prod_.words() + (size_t)k * ctw; };
    auto acc_at = [&](int which, int k) {
        return (which == 0 ? acc0_.words() : acc1_.words()) + (size_t)k * ctw;
    };
    auto acc_after = [&](int k, int done) -> u64* {  // accumulator after `done` doubling levels
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
    ORDER_ = put(order);
    PROD_ = put(vp);
    RLK_ = put(rlk);
    if (hoist) {
        std::vector<u64*> py(n);
        for (int k = 0; k < n; ++k)
            py[k] = (trees[order[k]].dbl.empty() && trees[order[k]].odd.empty()) ? nullptr : prodY_at(k);
        PRODY_ = put(py);
    }

    const bool fused = ctx.fused_key_switch();
    // the fused MAC also streams the key's Shoup companions
    const u64 C = sizeof(u64) * ctw, KEY = sizeof(u64) * ctx.ksk_words() * (fused ? 2 : 1),
              PT = sizeof(u64) * ctx.poly_words();
    stats_.chunks = n;
    stats_.slices = ns_;
    stats_.levels = depth;
    stats_.rotations = n_rot;
    stats_.hbm_bytes = n ? (u64)n * 3 * C + KEY : 0;
    stats_.key_bytes = n ? KEY : 0;
    // each NTT is two kernels (column, block phase); fused: extend, cols, blocks+tensor+iblocks,
    // icols, scale + the 4-kernel relinearisation key switch
    const bool ksc = std::getenv("CSSC_KS_CLUSTER") != nullptr;
    auto kfuse = [&](int items) { return fused && !ksc && ks_cols_moddown_applies(P, items) ? 1 : 0; };
    // multiply: extend, column phase, blocks + tensor, inverse columns, scale; the
    // relinearisation's key switch (4 launches, 3 with the fused finish) for the
    // products it is not folded into level 0 for
    const int n_relin = fold ? n - nd : n;
    stats_.kernels = n ? (fused ? 5 + (n_relin ? 4 - kfuse(n_relin) : 0) : 14) : 0;
    stats_.limb_ntts = (u64)n * (7 * M + P.dnum * LK + 2 * LK);  // + the rotate levels below

    std::set<u32> all_keys;
    u32 last_g = 0;
    auto key_of = [&](u64 offset, std::set<u32>& lvl, u32& gi) {
        const u32 g = galois_element((int64_t)offset, P.n);
        lvl.insert(g);
        all_keys.insert(g);
        gi = inverse_galois(g, P.n);
        last_g = g;
        return ctx.galois_key(g);
    };
    // level 0 rotates only products; with odd steps, several rotations share a
    // product: hoist its ModUp + forward NTT (CSSC_NO_HOIST=1 keeps per-item K1/K2)
    // Each odd step's key switch is summed into the doubling step it follows
    // (D_a, O_a share one INTT + ModDown; DESIGN 2.9, the oracle restates it):
    // level 0 accumulates every rotation of the products (doubling items
    // 0 .. nd-1, then the odd items: ACC[nd + o]), the odd items' c0 terms
    // phi_O(prod.c0) go to rp slot o (its c1 half stays zero) and are added as
    // EXTRA where their key switch is folded: level a-1 for O_a.
    const size_t accw = ctx.ksacc_words();
    std::vector<std::map<int, int>> odd_after(n);  // k -> (a -> odd slot o)
    std::vector<const u64*> odd_src;
    std::vector<u32> odd_gi;
    std::vector<u64*> odd_out;
    if (fold) {
        // stage slots: EXTRA (c0 terms: rp_ slot, c1 half zero) and bundle
        // (the stage's rotations of p, accumulated at level 0: ACC[nd + b])
        std::vector<std::vector<int>> xslot(n), bslot(n);
        int n_x = 0, n_b = 0;
        for (int k = 0; k < n; ++k) {
            const auto& sg = stages[order[k]];
            xslot[k].assign(sg.size(), -1);
            bslot[k].assign(sg.size(), -1);
            for (size_t t = 0; t < sg.size(); ++t) {
                if (!sg[t].poff.empty()) bslot[k][t] = n_b++;
                if (!sg[t].poff.empty() || sg[t].merged) xslot[k][t] = n_x++;
            }
        }
        auto xs_at = [&](int id) { return rp_.words() + (size_t)id * ctw; };
        const size_t pw2 = ctx.poly_words();
        int nt0 = 3;  // level 0's MAC terms per item: 3 per doubling item, 2 per bundled rotation of p
        for (int k = 0; k < n; ++k)
            for (const Stage& st : stages[order[k]]) nt0 = std::max(nt0, 2 * (int)st.poff.size());
        for (int l = 0; l < depth; ++l) {
            std::vector<const u64*> src, base, key, extra, ysrc, xacc, hp, hy, tk, asrc;
            std::vector<u64*> yout, o, aout;
            std::vector<u32> gi, tg, agi;
            std::vector<int> th;
            std::set<u32> lvl_keys;
            const int NT = l == 0 ? nt0 : 3;
            bool any_x = false, any_merged = false;
            auto term = [&](int h, u32 g, const u64* kp) {
                th.push_back(h);
                tg.push_back(g);
                tk.push_back(kp);
            };
            auto pad = [&](size_t upto) {
                while (th.size() < upto) term(-1, 1u, nullptr);
            };
            int tail = 0;
            for (int k = 0; k < n && (int)stages[order[k]].size() > l; ++k, ++tail) {
                const Stage& sg = stages[order[k]][l];
                u64* cur = acc_after(k, l);  // level 0: the product slot (z0, z1)
                u32 g;
                const u64* kd = key_of(sg.d1, lvl_keys, g);
                const u32 g1 = last_g;
                key.push_back(kd);
                gi.push_back(g);
                src.push_back(cur);
                base.push_back(cur);
                o.push_back(acc_at(l % 2, k));
                ysrc.push_back(yafter(k, l));
                yout.push_back((int)stages[order[k]].size() > l + 1 ? accY_at(l % 2, k) : nullptr);
                extra.push_back(xslot[k][l] >= 0 ? xs_at(xslot[k][l]) : nullptr);
                xacc.push_back(bslot[k][l] >= 0 ? ACC_.words() + (size_t)(nd + bslot[k][l]) * accw : nullptr);
                any_x = any_x || extra.back() || xacc.back();
                const size_t t0 = th.size();
                if (l == 0) {  // relinearisation of z2 + the rotation of z1 and z2
                    term(nd + k, 1u, ctx.relin_key());
                    term(k, g1, kd);
                    term(nd + k, g1, ctx.galois_key_sq(g1));
                } else {
                    term(k, g1, kd);
                    if (sg.merged) {  // R(acc, d2), R(acc, d1 + d2); their c0 terms into the EXTRA slot
                        any_merged = true;
                        aout.push_back(xs_at(xslot[k][l]));
                        for (u64 off : {sg.d2, sg.d1 + sg.d2}) {
                            u32 gx;
                            const u64* kx = key_of(off, lvl_keys, gx);
                            term(k, last_g, kx);
                            asrc.push_back(cur);
                            agi.push_back(gx);
                        }
                        asrc.push_back(nullptr);  // third term unused
                        agi.push_back(0);
                    }
                }
                pad(t0 + NT);
            }
            if (l == 0) {
                // the stages' rotations of p as level-0 bundle items, and every EXTRA
                // slot's c0 terms phi_o(z0) written (zero for merged-only slots)
                for (int k = 0; k < n; ++k) {
                    const auto& sg = stages[order[k]];
                    for (size_t t = 0; t < sg.size(); ++t) {
                        if (bslot[k][t] >= 0) {
                            const size_t t0 = th.size();
                            for (u64 off : sg[t].poff) {
                                u32 gx;
                                const u64* kx = key_of(off, lvl_keys, gx);
                                term(k, last_g, kx);
                                term(nd + k, last_g, ctx.galois_key_sq(last_g));
                            }
                            pad(t0 + NT);
                        }
                        if (xslot[k][t] >= 0) {
                            aout.push_back(xs_at(xslot[k][t]));
                            for (int x = 0; x < 3; ++x) {
                                const bool has = x < (int)sg[t].poff.size();
                                u32 gx = 0;
                                if (has) key_of(sg[t].poff[x], lvl_keys, gx);
                                asrc.push_back(has ? prod_at(k) : nullptr);
                                agi.push_back(has ? gx : 0u);
                            }
                        }
                    }
                }
            }
            Level lv;
            lv.items = tail;
            lv.acc_items = (int)(th.size() / NT);
            lv.src = put(src);
            lv.base = put(base);
            lv.out = put(o);
            lv.key = put(key);
            lv.ginv = put(gi);
            lv.extra = any_x ? put(extra) : nullptr;
            lv.xacc = any_x ? put(xacc) : nullptr;
            lv.ysrc = put(ysrc);
            lv.yout = put(yout);
            lv.pair = nullptr;
            lv.mac_terms = 0;
            for (int x : th) lv.mac_terms += x >= 0 ? 1 : 0;
            if (!aout.empty()) {
                lv.asum_n = (int)aout.size();
                lv.asum_out = put(aout);
                lv.asum_src = put(asrc);
                lv.asum_gi = put(agi);
                lv.asum_acc = l > 0;
            }
            if (l == 0 || any_merged) {  // hoisted: one ModUp + NTT per source, multi-term MAC
                if (l == 0) {  // sources: z1 of product k (c1 of its slot) -> H[k], z2 (D2) -> H[nd + k]
                    hp.resize(2 * nd);
                    hy.resize(2 * nd);
                    for (int k = 0; k < nd; ++k) {
                        hp[k] = prod_at(k) + pw2;
                        hy[k] = prodY_at(k);
                        hp[nd + k] = D2_.words() + (size_t)k * pw2;
                        hy[nd + k] = D2Y_.words() + (size_t)k * pw2;
                    }
                } else {  // sources: the accumulators' c1
                    hp.assign(src.begin(), src.end());
                    hy.assign(ysrc.begin(), ysrc.end());
                    for (auto& x : hp) x += pw2;
                }
                std::vector<int> ord(lv.acc_items);
                std::iota(ord.begin(), ord.end(), 0);
                if (std::getenv("CSSC_NO_KEY_ORDER") == nullptr)  // items sharing keys back to back (L2)
                    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) {
                        return tg[(size_t)x * NT + (l == 0 ? 1 : 0)] < tg[(size_t)y * NT + (l == 0 ? 1 : 0)];
                    });
                lv.horder = put(ord);
                lv.hsrc = (int)hp.size();
                lv.hprod = put(hp);
                lv.hy = put(hy);
                lv.hterm = NT;
                lv.hidx = put(th);
                lv.gel = put(tg);
                lv.hkey = put(tk);
            }
            lv.keys = (int)lvl_keys.size();
            levels_.push_back(lv);
            const int srcs = lv.hsrc ? lv.hsrc : lv.acc_items;
            const int kf = ks_cols_moddown_applies(P, lv.items) ? 1 : 0;
            stats_.hbm_bytes += (u64)lv.acc_items * 3 * C + lvl_keys.size() * KEY * (l == 0 ? 2 : 1);
            stats_.key_bytes += lvl_keys.size() * KEY * (l == 0 ? 2 : 1);
            stats_.kernels += 2 + (2 - kf) + (lv.hsrc ? 1 : 0) + (lv.asum_n ? 1 : 0);
            stats_.limb_ntts += (u64)srcs * P.dnum * LK + (u64)lv.items * 2 * LK;
        }
        if (n_x) cuda_check(cudaMemsetAsync(rp_.words(), 0, sizeof(u64) * ctw * n_x, ctx.stream()), "xs zero");
    } else {
    for (int l = 0; l < depth; ++l) {
        std::vector<const u64*> src, base, key, extra, ysrc, xacc;
        std::vector<u64*> yout;
        std::vector<u64*> o;
        std::vector<u32> gi, gel;
        std::vector<int> hidx;
        std::set<u32> lvl_keys;
        bool any_x = false;
        for (int k = 0; k < n && (int)trees[order[k]].dbl.size() > l; ++k) {
            const Tree& t = trees[order[k]];
            u64* cur = acc_after(k, l);
            u32 g;
            key.push_back(key_of(t.dbl[l], lvl_keys, g));
            gi.push_back(g);
            gel.push_back(last_g);
            hidx.push_back(k);
            src.push_back(cur);
            base.push_back(cur);
            o.push_back(acc_at(l % 2, k));
            ysrc.push_back(yafter(k, l));
            yout.push_back((int)t.dbl.size() > l + 1 ? accY_at(l % 2, k) : nullptr);
            extra.push_back(nullptr);
            xacc.push_back(nullptr);
        }
        const int tail = (int)o.size();
        if (l == 0) {  // the odd steps: rot(prod) of every chunk, accumulated in the same launch
            for (int k = 0; k < n; ++k) {
                for (const auto& [after, off] : trees[order[k]].odd) {
                    const int slot = (int)odd_src.size();
                    u32 g;
                    key.push_back(key_of(off, lvl_keys, g));
                    gi.push_back(g);
                    gel.push_back(last_g);
                    hidx.push_back(k);
                    src.push_back(prod_at(k));
                    ysrc.push_back(prodY_at(k));
                    odd_src.push_back(prod_at(k));
                    odd_gi.push_back(g);
                    odd_out.push_back(rp_.words() + (size_t)slot * ctw);
                    odd_after[k][after] = slot;
                }
            }
        }
        for (int k = 0; k < tail; ++k) {  // fold the odd step that follows D_{l+1}
            auto it = odd_after[k].find(l + 1);
            if (it == odd_after[k].end()) continue;
            extra[k] = rp_.words() + (size_t)it->second * ctw;
            xacc[k] = ACC_.words() + (size_t)(nd + it->second) * accw;
            any_x = true;
        }
        Level lv;
        lv.items = tail;
        lv.acc_items = (int)src.size();
        lv.mac_terms = lv.acc_items;
        lv.src = put(src);
        lv.base = put(base);
        lv.out = put(o);
        lv.key = put(key);
        lv.ginv = put(gi);
        lv.extra = any_x ? put(extra) : nullptr;
        lv.xacc = any_x ? put(xacc) : nullptr;
        lv.ysrc = hoist ? put(ysrc) : nullptr;
        lv.yout = hoist ? put(yout) : nullptr;
        lv.pair = nullptr;
        lv.keys = (int)lvl_keys.size();
        if (l == 0 && !odd_src.empty()) {
            lv.odd_n = (int)odd_src.size();
            lv.odd_src = put(odd_src);
            lv.odd_ginv = put(odd_gi);
            lv.odd_out = put(odd_out);
        }
        levels_.push_back(lv);
        const int srcs = lv.hsrc ? lv.hsrc : lv.acc_items;
        const int kf = fused && !ksc && ks_cols_moddown_applies(P, lv.items) ? 1 : 0;
        stats_.hbm_bytes += (u64)lv.acc_items * 3 * C + lvl_keys.size() * KEY;
        stats_.key_bytes += lvl_keys.size() * KEY;
        stats_.kernels += fused ? 2 + (2 - kf) + (any_x && !kf ? 1 : 0) + (lv.hsrc ? 1 : 0) + (lv.odd_n ? 1 : 0)
                                : 7 + (any_x ? 1 : 0) + (lv.odd_n ? 1 : 0);
        stats_.limb_ntts += (u64)srcs * P.dnum * LK + (u64)lv.items * 2 * LK;
    }
    }
    if (n_odd) cuda_check(cudaMemsetAsync(rp_.words(), 0, sizeof(u64) * ctw * n_odd, ctx.stream()), "rp zero");
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
        fin[k] = acc_after(k, (int)levels_of(order[k]));
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
    stats_.kernels += n ? (fused ? 3 : 5) : 0;
    stats_.limb_ntts += (u64)n * 2 * L + (u64)ns_ * 2 * L;
    if (!stage_.empty())
        cuda_check(cudaMemcpyAsync(arena_.as<void>(), stage_.data(), stage_.size(), cudaMemcpyHostToDevice,
                                   ctx.stream()),
                   "plan upload");
    ctx.synchronize();
}

CloudPlan::~CloudPlan() {
    if (pexec_) cudaGraphExecDestroy(pexec_);
    if (eexec_) cudaGraphExecDestroy(eexec_);
    if (ev_early_) cudaEventDestroy(ev_early_);
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (exec_) cudaGraphExecDestroy(exec_);
    if (graph_) cudaGraphDestroy(graph_);
}

void CloudPlan::record(std::vector<cudaEvent_t>* marks, u64* dec_d, const EncIn* enc) {
    if (n_ == 0) return;
    const RnsParams& P = ctx_.params();
    const int L = P.cfg.L, logn = P.cfg.logn;
    cudaStream_t st = ctx_.stream();
    auto mark = [&] {
        kmark("@group", st);
        if (!marks) return;
        cudaEvent_t e;
        cuda_check(cudaEventCreate(&e), "event");
        // External: under stream capture this becomes an event-record node
        cuda_check(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal), "event record");
        marks->push_back(e);
    };
    mark();
    {
        const NvtxRange nv("cssc.cloud.multiply");
        ctx_.mul_relin_dev(A_, B_, PROD_, n_, T_.words(), Z_.words(), D2_.words(), DX_.words(),
                           ACC_.words(), RLK_, enc, PRODY_ ? D2Y_.words() : nullptr, PRODY_, fold_ ? nd_ : 0,
                           fold_ ? PRODY_ : nullptr);
    }
    mark();
    const bool fused = ctx_.fused_key_switch();
    for (size_t l = 0; l < levels_.size(); ++l) {
        const NvtxRange nv("cssc.cloud.key_switch_stage");
        const Level& lv = levels_[l];
        KsY ky;
        ky.src = lv.ysrc;
        HoistedKs hk;
        if (lv.hsrc) {
            hk.nsrc = lv.hsrc;
            hk.src = lv.hprod;
            hk.src_poly = 0;
            hk.ysrc = lv.hy;
            hk.nterm = lv.hterm;
            hk.hidx = lv.hidx;
            hk.gel = lv.gel;
            hk.order = lv.horder;
        }
        const KsAccDomain dom = launch_ks_accumulate(ctx_.dconsts(), P, fused, lv.src, lv.ginv,
                                                     lv.hsrc ? lv.hkey : lv.key, DX_.words(), ACC_.words(),
                                                     lv.acc_items, st, ky, lv.hsrc ? &hk : nullptr);
        if (lv.odd_n) {
            launch_automorph_c0(ctx_.dconsts(), P, lv.odd_src, lv.odd_ginv, lv.odd_out, lv.odd_n, st);
            kmark("k_automorph_c0", st);
        }
        if (lv.asum_n) {
            launch_automorph_sum(ctx_.dconsts(), P, lv.asum_out, lv.asum_src, lv.asum_gi, lv.asum_acc, lv.asum_n, st);
            kmark("k_automorph_sum", st);
        }
        launch_ks_finish(ctx_.dconsts(), P, dom, lv.base, lv.src, lv.ginv, lv.out, ACC_.words(), lv.items, st,
                         lv.extra, lv.yout, lv.xacc);
        mark();
    }
    const NvtxRange nv_mask("cssc.cloud.mask_sum");
    std::vector<int> qidx(L);
    std::iota(qidx.begin(), qidx.end(), 0);
    NttJob fwd = ctx_.job(nullptr, MT_.words(), 2 * L, qidx);
    fwd.src_items = FINAL_;
    NttJob inv = ctx_.job(nullptr, nullptr, 2 * L, qidx);
    inv.dst_items = OUT_;
    if (dec_d) {  // column phase, fused blocks + mask MAC + (c0 + c1 s) + inverse blocks
        launch_ntt_phase(ctx_.dconsts(), logn, false, true, fwd, n_, st);
        launch_mask_dec_blocks(ctx_.dconsts(), P, MT_.words(), slice_off_, slice_items_, item_mask_,
                               MASKS_.words(), ctx_.s_ntt(), dec_d, ns_, st);
    } else if (ctx_.fused_key_switch()) {  // column phase, fused blocks + mask MAC + inverse blocks, column phase
        launch_ntt_phase(ctx_.dconsts(), logn, false, true, fwd, n_, st);
        kmark("k_ntt_cols fwd (mask)", st);
        launch_mask_blocks(ctx_.dconsts(), P, MT_.words(), slice_off_, slice_items_, item_mask_, MASKS_.words(),
                           OUT_, ns_, st);
        kmark("k_mask_blocks", st);
        launch_ntt_phase(ctx_.dconsts(), logn, true, true, inv, ns_, st);
        kmark("k_ntt_cols inv (mask)", st);
    } else {
        launch_ntt(ctx_.dconsts(), logn, false, fwd, n_, st);
        u64* RES = T_.words();  // ns <= n results fit the multiply workspace
        launch_mask_accum(ctx_.dconsts(), P, MT_.words(), slice_off_, slice_items_, item_mask_,
                          MASKS_.words(), RES, ns_, st);
        inv.src = RES;
        launch_ntt(ctx_.dconsts(), logn, true, inv, ns_, st);
    }
    mark();
}

std::vector<PhaseTiming> CloudPlan::profile() {
    std::vector<PhaseTiming> out;
    if (n_ == 0) return out;
    const RnsParams& P = ctx_.params();
    const int L = P.cfg.L, LK = L + P.cfg.K, M = P.mul_limbs();
    const u64 C = sizeof(u64) * ctx_.ct_words(),
              KEY = sizeof(u64) * ctx_.ksk_words() * (ctx_.fused_key_switch() ? 2 : 1),
              PT = sizeof(u64) * ctx_.poly_words();
    const u64 ks_ntts = (u64)P.dnum * LK + 2 * LK;
    const u64 nrel = (u64)(n_ - (fold_ ? nd_ : 0));  // relinearised products (the rest fold into level 0)
    out.push_back({"multiply+relin", 0, (u64)n_, (u64)n_ * 3 * C + (nrel ? KEY : 0), (u64)n_ * 7 * M + nrel * ks_ntts,
                   nrel, nrel, nrel});
    for (size_t l = 0; l < levels_.size(); ++l) {
        const Level& lv = levels_[l];
        const u64 srcs = lv.hsrc ? (u64)lv.hsrc : (u64)lv.acc_items;
        out.push_back({"rotate level " + std::to_string(l), 0, (u64)lv.items,
                       (u64)lv.acc_items * 3 * C + (u64)lv.keys * KEY,
                       srcs * P.dnum * LK + (u64)lv.items * 2 * LK, srcs, (u64)lv.acc_items,
                       (u64)lv.mac_terms});
    }
    out.push_back({"mask accumulate", 0, (u64)n_, (u64)n_ * 2 * C + (u64)n_masks_ * PT,
                   (u64)n_ * 2 * L + (u64)ns_ * 2 * L, (u64)n_, (u64)n_, 0});
    // captured like run(), with event-record nodes between the groups, so the
    // timings include the graph's (small) inter-kernel gaps and nothing else
    std::vector<cudaEvent_t> marks;
    cudaStream_t st = ctx_.stream();
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ex = nullptr;
    try {
        cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
        try {
            record(&marks);
        } catch (...) {
            cudaGraph_t tmp = nullptr;
            cudaStreamEndCapture(st, &tmp);
            if (tmp) cudaGraphDestroy(tmp);
            throw;
        }
        cuda_check(cudaStreamEndCapture(st, &g), "end capture");
        cuda_check(cudaGraphInstantiate(&ex, g, 0), "graph instantiate");
        cuda_check(cudaGraphUpload(ex, st), "graph upload");
        cuda_check(cudaGraphLaunch(ex, st), "graph launch");
        cuda_check(cudaStreamSynchronize(st), "profile");
    } catch (...) {
        if (ex) cudaGraphExecDestroy(ex);
        if (g) cudaGraphDestroy(g);
        for (auto e : marks) cudaEventDestroy(e);
        throw;
    }
    cudaGraphExecDestroy(ex);
    cudaGraphDestroy(g);
    for (size_t i = 0; i + 1 < marks.size() && i < out.size(); ++i) {
        float ms = 0;
        const cudaError_t e = cudaEventElapsedTime(&ms, marks[i], marks[i + 1]);
        if (e != cudaSuccess) {
            for (auto m : marks) cudaEventDestroy(m);
            cuda_check(e, "profile event timing");
        }
        out[i].us = 1e3 * ms;
    }
    for (auto e : marks) cudaEventDestroy(e);
    return out;
}

std::vector<KernelTiming> CloudPlan::profile_kernels(int reps, size_t flush_bytes) {
    std::vector<KernelTiming> out;
    if (n_ == 0 || reps < 1) return out;
    cudaStream_t st = ctx_.stream();
    std::vector<KernelMark> km;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ex = nullptr;
    auto cleanup = [&] {
        kmarks_install(nullptr);
        if (ex) cudaGraphExecDestroy(ex);
        if (g) cudaGraphDestroy(g);
        for (auto& m : km) cudaEventDestroy(m.ev);
    };
    try {
        DevBuf flush(&ctx_.pool(), flush_bytes ? flush_bytes : 8);
        kmarks_install(&km);
        cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
        try {
            record();
        } catch (...) {
            cudaGraph_t tmp = nullptr;
            cudaStreamEndCapture(st, &tmp);
            if (tmp) cudaGraphDestroy(tmp);
            throw;
        }
        kmarks_install(nullptr);
        cuda_check(cudaStreamEndCapture(st, &g), "end capture");
        cuda_check(cudaGraphInstantiate(&ex, g, 0), "graph instantiate");
        cuda_check(cudaGraphUpload(ex, st), "graph upload");
        int group = 0;
        for (size_t i = 1; i < km.size(); ++i) {
            if (std::strcmp(km[i].name, "@group") == 0)
                ++group;
            else
                out.push_back({km[i].name, group, 0.0});
        }
        for (int r = 0; r < reps; ++r) {
            if (flush_bytes) cuda_check(cudaMemsetAsync(flush.words(), r & 0xff, flush_bytes, st), "flush");
            cuda_check(cudaGraphLaunch(ex, st), "graph launch");
            cuda_check(cudaStreamSynchronize(st), "profile kernels");
            size_t k = 0;
            for (size_t i = 1; i < km.size(); ++i) {
                float ms = 0;
                cuda_check(cudaEventElapsedTime(&ms, km[i - 1].ev, km[i].ev), "profile event timing");
                if (std::strcmp(km[i].name, "@group") != 0) out[k++].us += 1e3 * ms / reps;
            }
        }
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
    return out;
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

namespace cssc {

void CloudPlan::capture_pipeline(const unsigned char* img, const CsscLayout& lay, unsigned char* out) {
    if (n_ == 0) throw std::invalid_argument("pipeline: empty plan");
    if (lay.items != 2 * n_) throw std::invalid_argument("pipeline: image does not match the plan's chunks");
    if (pexec_) {
        cudaGraphExecDestroy(pexec_);
        pexec_ = nullptr;
    }
    if (eexec_) {
        cudaGraphExecDestroy(eexec_);
        eexec_ = nullptr;
    }
    const RnsParams& P = ctx_.params();
    const size_t n = (size_t)P.n, L = (size_t)P.cfg.L;
    DevicePool* pool = &ctx_.pool();
    pup_.ensure(pool, std::max<size_t>(lay.bytes, 256));
    pU_.ensure(pool, sizeof(u64) * (size_t)lay.items * L * n);
    pCM_.ensure(pool, sizeof(u64) * (size_t)lay.items * ctx_.cm_stride());
    pX_.ensure(pool, sizeof(u64) * (size_t)ns_ * L * n);
    pM_.ensure(pool, sizeof(u64) * (size_t)ns_ * n);
    pslots_.ensure(pool, pipeline_out_bytes() + 64);
    pE_.ensure(pool, (size_t)lay.items * 2 * n);
    {
        std::vector<int> g(2 * (size_t)ns_);
        for (int s2 = 0; s2 < ns_; ++s2) {
            g[s2] = rows_[s2];
            g[ns_ + s2] = (int)out_off_[s2];
        }
        pgather_.ensure(pool, sizeof(int) * std::max<size_t>(g.size(), 1));
        cuda_check(cudaMemcpy(pgather_.as<int>(), g.data(), sizeof(int) * g.size(), cudaMemcpyHostToDevice),
                   "gather table");
    }
    ClientWs ws;
    ws.up = pup_.as<unsigned char>();
    ws.U = pU_.words();
    ws.CM = pCM_.words();
    ws.X = pX_.words();
    ws.M = pM_.words();
    ws.slots = pslots_.words();
    ws.E = pE_.as<int8_t>();
    auto* maxdev = reinterpret_cast<unsigned long long*>(pslots_.as<unsigned char>() + maxdev_off_);
    cudaStream_t st = ctx_.stream();
    cudaGraph_t g = nullptr;
    static const bool prof = std::getenv("CSSC_PIPE_PROFILE") != nullptr;
    for (cudaEvent_t ev : pmarks_) cudaEventDestroy(ev);
    pmarks_.clear();
    std::vector<cudaEvent_t>* mk = prof ? &pmarks_ : nullptr;
    auto mark = [&] {
        if (!mk) return;
        cudaEvent_t ev;
        cuda_check(cudaEventCreate(&ev), "event");
        cuda_check(cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal), "event record");
        mk->push_back(ev);
    };
    if (!ev_early_) cuda_check(cudaEventCreateWithFlags(&ev_early_, cudaEventDisableTiming), "event");
    if (!ev_fork_) cuda_check(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming), "event");
    {  // early graph: the encryption's message-independent branch
        cudaGraph_t ge = nullptr;
        cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
        try {
            ctx_.encrypt_cssc_image(img, lay, &ws, nullptr, 1);
        } catch (...) {
            cudaGraph_t tmp = nullptr;
            cudaStreamEndCapture(st, &tmp);
            if (tmp) cudaGraphDestroy(tmp);
            throw;
        }
        cuda_check(cudaStreamEndCapture(st, &ge), "end capture");
        const cudaError_t e = cudaGraphInstantiate(&eexec_, ge, 0);
        cudaGraphDestroy(ge);
        cuda_check(e, "graph instantiate");
    }
    cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
        mark();
        // fused path: the encryption's finish rides in the multiply's base
        // extension, the decryption in the mask step (k_mask_dec_blocks)
        const int fuse_mask = ctx_.pipe_fuse();  // bit 0 encryption finish, bit 1 decryption
        const bool fused = ctx_.fused_key_switch() && fixed_rns_shape(P);
        const bool fenc = fused && (fuse_mask & 1), fdec = fused && (fuse_mask & 2);
        EncIn enc{};
        ctx_.encrypt_cssc_image(img, lay, &ws, fenc ? &enc : nullptr, 2, ev_early_);
        enc.order = ORDER_;  // the multiply's items are the chunks in depth order
        const int* grows = pgather_.as<int>();
        if (fdec) {
            record(mk, ws.X, fenc ? &enc : nullptr);
            launch_decrypt_ntt(ctx_.dconsts(), P, ws.X, ws.M, nullptr, maxdev, ns_, st);
        } else {
            record(mk, nullptr, fenc ? &enc : nullptr);
            ctx_.decrypt_dev(OUT_, ns_, ws.X, ws.M, nullptr, maxdev);
        }
        int rmax = 0;
        for (int v : rows_) rmax = std::max(rmax, v);
        launch_decode_rows(ctx_.dconsts(), P, ws.M, reinterpret_cast<u32*>(ws.slots), grows, grows + ns_, rmax,
                           ns_, st);
        mark();
        cuda_check(cudaMemcpyAsync(out, ws.slots, pipeline_out_bytes(), cudaMemcpyDeviceToHost, st), "download");
        mark();
    } catch (...) {
        cudaGraph_t tmp = nullptr;
        cudaStreamEndCapture(st, &tmp);
        if (tmp) cudaGraphDestroy(tmp);
        throw;
    }
    cuda_check(cudaStreamEndCapture(st, &g), "end capture");
    const cudaError_t e = cudaGraphInstantiate(&pexec_, g, 0);
    cudaGraphDestroy(g);
    cuda_check(e, "graph instantiate");
}

// The early graph runs on the side stream (after everything already on the
// context stream); the main graph's image branch starts beside it and its
// join waits for ev_early_ (an external event-wait node).
void CloudPlan::run_early() {
    if (!eexec_) throw std::logic_error("pipeline not captured");
    cudaStream_t side = ctx_.side_stream();
    cuda_check(cudaEventRecord(ev_fork_, ctx_.stream()), "fork");
    cuda_check(cudaStreamWaitEvent(side, ev_fork_, 0), "fork");
    cuda_check(cudaGraphLaunch(eexec_, side), "graph launch");
    cuda_check(cudaEventRecord(ev_early_, side), "event record");
}

void CloudPlan::run_pipeline(bool early_done) {
    if (!pexec_) throw std::logic_error("pipeline not captured");
    if (!early_done) run_early();
    cuda_check(cudaGraphLaunch(pexec_, ctx_.stream()), "graph launch");
    if (!pmarks_.empty()) {  // CSSC_PIPE_PROFILE: encrypt | multiply | levels.. | mask | decrypt | download
        cuda_check(cudaStreamSynchronize(ctx_.stream()), "sync");
        std::fprintf(stderr, "pipe-profile us:");
        for (size_t i = 1; i < pmarks_.size(); ++i) {
            float ms = 0;
            cudaEventElapsedTime(&ms, pmarks_[i - 1], pmarks_[i]);
            std::fprintf(stderr, " %.1f", 1e3 * ms);
        }
        std::fprintf(stderr, "\n");
    }
}

}  // namespace cssc
