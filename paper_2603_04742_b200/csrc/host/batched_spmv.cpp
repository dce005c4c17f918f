// batched_spmv.cpp -- see batched_spmv.hpp.
#include "batched_spmv.hpp"

#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <exception>
#include <climits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>

#include "host/host_pool.hpp"
#include "nvtx_range.hpp"
#include "spmv/gpu_backend.hpp"

namespace spmv::detail {

namespace {

// reference protocol.cpp:108-111: a 4-byte count, then an (h, k) header and
// 4-byte indices for every padded slot of every chunk
std::uint64_t column_index_bytes(const std::uint64_t* r, const std::uint64_t* c, std::size_t n) {
    std::uint64_t b = 4;
    for (std::size_t i = 0; i < n; ++i) b += 8 + 4 * r[i] * c[i];
    return b;
}

int lowered(int b, int c) { return std::max(0, b - c); }

// batches with at least this many nonzeros use the host pool for the CSR
// scans and the pinned image (C2's 16 777 stay single-threaded)
constexpr std::size_t kParallelEntries = 1 << 18;

}  // namespace

CsrView view_of(const CsrMatrix& m, std::span<const std::int64_t> v) {
    if (m.cols != v.size())
        throw DimensionMismatchError("spmv_partitioned: vector length does not match columns");
    if (m.row_ptrs.size() != m.rows + 1 || m.col_indices.size() != m.values.size())
        throw std::invalid_argument("csr: inconsistent array lengths");
    CsrView w;
    w.rows = m.rows;
    w.cols = m.cols;
    w.nnz = m.values.size();
    w.row_ptrs = reinterpret_cast<const std::uint64_t*>(m.row_ptrs.data());
    w.col_indices = reinterpret_cast<const std::uint64_t*>(m.col_indices.data());
    w.values = m.values.data();
    w.vec = v.data();
    return w;
}

BatchedSpmv::BatchedSpmv(spmvgpu_ctx* ctx, const HeParams& hp, std::span<const CsrView> ms,
                         std::size_t chunk_size, PartyRole key_holder, bool partition, int rank, int world)
    : ctx_(ctx), hp_(hp), kh_(key_holder), nmat_(ms.size()), rank_(rank), world_(world) {
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("shard: rank must be in [0, world)");
    const cssc::NvtxRange nvtx_("cssc.pack");
    static const bool trace = std::getenv("CSSC_TRACE_E2E") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    std::size_t nnz_total = 0, vec_total = 0;
    for (const CsrView& m : ms) {
        nnz_total += m.nnz;
        vec_total += m.cols;
    }
    if (nnz_total > INT32_MAX || vec_total > INT32_MAX)
        throw std::length_error("spmv_batch: more than 2^31 entries in one batch");
    // large batches: the row_ptrs scan runs on the host pool; the column-range
    // check rides in the image pass below (one read of the column indices).
    // Any failure re-runs the checks in the reference's order (raise_first).
    const bool big = nnz_total >= kParallelEntries;
    bool rows_ok = false;
    // the compact client image: int8 values / vector entries when all fit,
    // 16-bit column indices when every matrix has at most 2^16 columns
    bool va_narrow = true, v_narrow = true;
    if (big) {
        constexpr std::size_t kBlock = 1 << 16;
        std::vector<std::pair<std::size_t, std::size_t>> tasks;  // (matrix, block of rows)
        for (std::size_t mi = 0; mi < ms.size(); ++mi)
            for (std::size_t b0 = 0; b0 * kBlock < ms[mi].rows; ++b0) tasks.push_back({mi, b0});
        std::vector<unsigned char> bad(tasks.size(), 0);
        HostPool::get().run(tasks.size(), [&](std::size_t t) {
            const CsrView& m = ms[tasks[t].first];
            const std::size_t b0 = tasks[t].second * kBlock;
            bool dec = false;
            for (std::size_t i = b0; i < std::min(m.rows, b0 + kBlock); ++i) dec |= m.row_ptrs[i + 1] < m.row_ptrs[i];
            bad[t] = dec;
        });
        rows_ok = std::none_of(bad.begin(), bad.end(), [](unsigned char x) { return x != 0; });
        // values: int8 assumed, checked while the image is written (one pass over them)
    } else {
        for (const CsrView& m : ms) {
            std::uint64_t outside8 = 0;
            for (std::size_t k = 0; k < m.nnz; ++k) outside8 |= (static_cast<std::uint64_t>(m.values[k]) + 128) >> 8;
            va_narrow = va_narrow && outside8 == 0;
        }
    }
    std::size_t max_cols = 0;
    for (const CsrView& m : ms) {
        max_cols = std::max(max_cols, m.cols);
        std::uint64_t outside8 = 0;
        for (std::size_t k = 0; k < m.cols; ++k) outside8 |= (static_cast<std::uint64_t>(m.vec[k]) + 128) >> 8;
        v_narrow = v_narrow && outside8 == 0;
    }
    // all col < cols: every col - cols is negative (and no col has bit 63 set)
    auto cols_in_range = [](const CsrView& m, std::size_t k0, std::size_t k1) {
        std::uint64_t all_neg = ~std::uint64_t{0}, any_top = 0;
        for (std::size_t k = k0; k < k1; ++k) {
            all_neg &= m.col_indices[k] - m.cols;
            any_top |= m.col_indices[k];
        }
        return k0 >= k1 || ((all_neg >> 63) && !(any_top >> 63));
    };
    auto col_check = [&](const CsrView& m) {  // branch-free scan; the offending entry is located only on failure
        if (cols_in_range(m, 0, m.nnz)) return;
        for (std::size_t k = 0; k < m.nnz; ++k)
            if (m.col_indices[k] >= m.cols)
                throw IndexOutOfRangeError("csr: column index " + std::to_string(m.col_indices[k]) +
                                           " out of range for " + std::to_string(m.cols) + " columns");
    };
    // validation in matrix order; the slices to shape are collected and shaped
    // afterwards (on the host pool for large batches), errors still surface in
    // the order the sequential evaluation would raise them
    const auto tv = std::chrono::steady_clock::now();
    std::vector<SliceJob> jobs;
    std::exception_ptr pending;
    std::size_t fail_mat = ms.size();
    bool pending_after_cols = false;  // the failed check comes after the matrix's column check
    std::int64_t nz_next = 0, vec_next = 0;
    for (std::size_t mi = 0; mi < ms.size() && !pending; ++mi) {
        bool past_cols = false;
        try {
            const CsrView& m = ms[mi];
            if (m.rows && m.row_ptrs[0] != 0) throw std::invalid_argument("csr: row_ptrs[0] must be 0");
            if (!rows_ok) {
                bool dec = false;
                for (std::size_t i = 0; i < m.rows; ++i) dec |= m.row_ptrs[i + 1] < m.row_ptrs[i];
                if (dec) throw std::invalid_argument("csr: row_ptrs must be non-decreasing");
            }
            if (m.rows && m.row_ptrs[m.rows] != m.nnz) throw std::invalid_argument("csr: row_ptrs end is not nnz");
            if (!big) col_check(m);
            past_cols = true;
            const std::int64_t nz_base = nz_next, vec_base = vec_next;
            nz_next += static_cast<std::int64_t>(m.nnz);
            vec_next += static_cast<std::int64_t>(m.cols);
            rows_of_.push_back(m.rows);
            // spmv_partitioned slices rows by chunk_size (partition_rows, chunk.cpp:55-73);
            // plain spmv keeps one slice
            if (partition) {
                if (chunk_size == 0) throw std::invalid_argument("partition_rows: max_rows must be positive");
                for (std::size_t r0 = 0; r0 < m.rows; r0 += chunk_size)
                    jobs.push_back({mi, r0, std::min(m.rows, r0 + chunk_size), nz_base, vec_base});
            } else {
                jobs.push_back({mi, 0, m.rows, nz_base, vec_base});
            }
        } catch (...) {
            pending = std::current_exception();
            fail_mat = mi;
            pending_after_cols = past_cols;
        }
    }
    std::vector<SliceShape> shapes(jobs.size());
    {
        auto shape_one = [&](std::size_t j) {
            try {
                shape_slice(ms[jobs[j].mat], jobs[j], chunk_size, shapes[j]);
            } catch (...) {
                shapes[j].err = std::current_exception();
            }
        };
        const auto tj = std::chrono::steady_clock::now();
        if (big && jobs.size() > 1)
            HostPool::get().run(jobs.size(), shape_one);
        else
            for (std::size_t j = 0; j < jobs.size(); ++j) shape_one(j);
        if (trace) {
            auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
            std::fprintf(stderr, "e2e-trace scan %.1f validate %.1f shape %.1f us\n", us(t0, tv), us(tv, tj),
                         us(tj, std::chrono::steady_clock::now()));
        }
    }
    // the first error in the reference's order: per matrix its CSR checks (the
    // column check deferred for large batches), then its slices' shape errors;
    // with no earlier error, the failed matrix's own checks
    auto raise_first = [&] {
        std::size_t j = 0;
        for (std::size_t mi = 0; mi < fail_mat; ++mi) {
            if (big) col_check(ms[mi]);
            for (; j < jobs.size() && jobs[j].mat == mi; ++j)
                if (shapes[j].err) std::rethrow_exception(shapes[j].err);
        }
        if (pending) {
            if (big && pending_after_cols) col_check(ms[fail_mat]);
            std::rethrow_exception(pending);
        }
    };
    if (pending || std::any_of(shapes.begin(), shapes.end(), [](const SliceShape& s) { return bool(s.err); }))
        raise_first();
    const auto ts = std::chrono::steady_clock::now();
    // slice metadata in order; the row / column records are written straight
    // into the image below, each slice's at its offsets computed here
    std::vector<std::size_t> row_at(jobs.size() + 1, 0), col_at(jobs.size() + 1, 0);
    std::vector<std::int64_t> nz_at(jobs.size() + 1, 0);  // rpre base: entries of the earlier slices
    std::vector<std::int32_t> chunk0(jobs.size()), sidx(jobs.size());
    for (std::size_t j = 0; j < jobs.size(); ++j) {
        const CsrView& m = ms[jobs[j].mat];
        row_at[j + 1] = row_at[j] + shapes[j].rowrec.size() / 4;
        col_at[j + 1] = col_at[j] + shapes[j].colrec.size() / 4;
        nz_at[j + 1] = nz_at[j] + static_cast<std::int64_t>(m.row_ptrs[jobs[j].r1] - m.row_ptrs[jobs[j].r0]);
        chunk0[j] = static_cast<std::int32_t>(r_.size());
        sidx[j] = static_cast<std::int32_t>(slicerec_.size() / 2);
        append_slice(shapes[j], col_at[j]);
    }
    // this rank's chunks (round-robin over global chunk indices);
    // world == 1 keeps every chunk
    std::vector<std::int32_t> local_of(r_.size(), -1);
    res_local_.assign(n_out_, -1);
    for (std::size_t g = 0; g < r_.size(); ++g) {
        if ((int)(g % (std::size_t)world_) != rank_) continue;
        local_of[g] = static_cast<std::int32_t>(dr_.size());
        dr_.push_back(r_[g]);
        dc_.push_back(c_[g]);
        const std::uint32_t res = slice_id_[g];
        if (res_local_[res] < 0) res_local_[res] = static_cast<int>(n_dout_++);
        dslice_.push_back(static_cast<std::uint32_t>(res_local_[res]));
    }
    const std::size_t n = dr_.size();
    if (!n) {  // no image: the deferred column checks on their own
        if (big)
            for (const CsrView& m : ms) col_check(m);
        return;
    }
    // the cloud's view of the job: chunk shapes and slice ids (ChunkShapeMeta)
    std::vector<std::uint64_t> key{n, n_dout_};
    key.insert(key.end(), dr_.begin(), dr_.end());
    key.insert(key.end(), dc_.begin(), dc_.end());
    key.insert(key.end(), dslice_.begin(), dslice_.end());
    const auto t1 = std::chrono::steady_clock::now();
    const bool hit = plan_cache_take(ctx_, key, lease_);
    // the client upload image, written once straight from the callers' arrays
    // and the slice shapes: into the cached pipeline's own pinned buffer when
    // its layout matches
    const int ci_w = max_cols <= (std::size_t{1} << 16) ? 2 : 4, v_w = v_narrow ? 1 : 8;
    const auto t1b = std::chrono::steady_clock::now();
    // narrowing copies of the column indices (range-checked for large batches),
    // values (int8 checked) and vectors
    enum Narrow { CI16, CI32, I8, I8V, I64 };
    struct Piece {
        unsigned char* d;
        const void* src;
        std::size_t cnt;
        Narrow kind;
        const CsrView* m;  // column pieces of large batches: the matrix to range-check against
    };
    // false when a value did not fit (I8V) or a column was out of range
    auto narrow = [&](const Piece& p) -> bool {
        switch (p.kind) {
            case CI16:
            case CI32: {
                const auto* x = static_cast<const std::uint64_t*>(p.src);
                std::uint64_t all_neg = ~std::uint64_t{0}, any_top = 0;
                const std::uint64_t cols = p.m ? p.m->cols : 0;
                if (p.kind == CI16) {
                    auto* o = reinterpret_cast<std::uint16_t*>(p.d);
                    for (std::size_t i = 0; i < p.cnt; ++i) {
                        o[i] = static_cast<std::uint16_t>(x[i]);
                        all_neg &= x[i] - cols;
                        any_top |= x[i];
                    }
                } else {
                    auto* o = reinterpret_cast<std::uint32_t*>(p.d);
                    for (std::size_t i = 0; i < p.cnt; ++i) {
                        o[i] = static_cast<std::uint32_t>(x[i]);
                        all_neg &= x[i] - cols;
                        any_top |= x[i];
                    }
                }
                return !p.m || p.cnt == 0 || ((all_neg >> 63) && !(any_top >> 63));
            }
            case I8:
            case I8V: {
                auto* o = reinterpret_cast<std::int8_t*>(p.d);
                const auto* x = static_cast<const std::int64_t*>(p.src);
                std::uint64_t outside8 = 0;
                for (std::size_t i = 0; i < p.cnt; ++i) {
                    o[i] = static_cast<std::int8_t>(x[i]);
                    outside8 |= (static_cast<std::uint64_t>(x[i]) + 128) >> 8;  // outside [-128, 127]
                }
                return outside8 == 0;
            }
            case I64:
                if (p.cnt) std::memcpy(p.d, p.src, 8 * p.cnt);
                return true;
        }
        return true;
    };
    double t_place = 0;
    // returns {values fit the image's width, columns in range}
    auto build_image = [&](int va_w) -> std::pair<bool, bool> {
        ClientImage lay = client_image_layout(nnz_total, vec_total, row_at.back(), slicerec_.size() / 2,
                                              col_at.back(), static_cast<int>(2 * n), ci_w, va_w, v_w);
        if (hit && lease_.pimg && lease_.pkey == client_image_key(lay)) {
            img_ = lay;
            img_.p = lease_.pimg;
            img_.cap = lease_.pimg_cap;
            img_borrowed_ = true;
        } else {
            img_ = client_image_take(ctx_, nnz_total, vec_total, row_at.back(), slicerec_.size() / 2,
                                     col_at.back(), static_cast<int>(2 * n), ci_w, va_w, v_w);
            img_borrowed_ = false;
        }
        const auto tp = std::chrono::steady_clock::now();
        std::vector<Piece> pieces;
        constexpr std::size_t kElems = 1 << 16;
        auto add = [&](unsigned char* d, std::size_t dw, const void* src, std::size_t cnt, Narrow kind,
                       const CsrView* m) {
            for (std::size_t o = 0; o < cnt; o += kElems)
                pieces.push_back({d + dw * o, static_cast<const std::uint64_t*>(src) + o, std::min(kElems, cnt - o),
                                  kind, m});
        };
        std::size_t nz = 0, vo = 0;
        for (const CsrView& m : ms) {
            add(img_.p + img_.o_ci + (std::size_t)img_.ci_w * nz, img_.ci_w, m.col_indices, m.nnz,
                img_.ci_w == 2 ? CI16 : CI32, big ? &m : nullptr);
            add(img_.p + img_.o_va + (std::size_t)img_.va_w * nz, img_.va_w, m.values, m.nnz,
                img_.va_w == 1 ? I8V : I64, nullptr);
            add(img_.p + img_.o_v + (std::size_t)img_.v_w * vo, img_.v_w, m.vec, m.cols, img_.v_w == 1 ? I8 : I64,
                nullptr);
            nz += m.nnz;
            vo += m.cols;
        }
        if (!slicerec_.empty()) std::memcpy(img_.p + img_.o_sl, slicerec_.data(), 4 * slicerec_.size());
        auto* rows = reinterpret_cast<std::int32_t*>(img_.p + img_.o_rows);
        auto* pre = reinterpret_cast<std::int32_t*>(img_.p + img_.o_rpre);
        auto* cols = reinterpret_cast<std::int32_t*>(img_.p + img_.o_cols);
        pre[row_at.back()] = static_cast<std::int32_t>(nz_at.back());
        // slice j's device records {nz_begin, len, pos, slice} and the exclusive
        // prefix of the row lengths (the device pack's entry -> row map), and its
        // column records {local chunk, k, h, 0}
        auto place = [&](std::size_t j) {
            const SliceShape& sh = shapes[j];
            std::int32_t* rr = rows + 4 * row_at[j];
            std::int32_t* rp = pre + row_at[j];
            std::int32_t acc = static_cast<std::int32_t>(nz_at[j]);
            for (std::size_t i = 0, r = 0; i < sh.rowrec.size(); i += 4, ++r) {
                rr[i] = sh.rowrec[i];
                rr[i + 1] = sh.rowrec[i + 1];
                rr[i + 2] = sh.rowrec[i + 2];
                rr[i + 3] = sidx[j];
                rp[r] = acc;
                acc += sh.rowrec[i + 1];
            }
            std::int32_t* cr = cols + 4 * col_at[j];
            for (std::size_t i = 0; i < sh.colrec.size(); i += 4) {
                cr[i] = local_of[static_cast<std::size_t>(sh.colrec[i] + chunk0[j])];
                cr[i + 1] = sh.colrec[i + 1];
                cr[i + 2] = sh.colrec[i + 2];
                cr[i + 3] = sh.colrec[i + 3];
            }
        };
        const std::size_t ns = slices_.size(), np = pieces.size();
        std::vector<unsigned char> miss(np, 0);
        auto task = [&](std::size_t i) {
            if (i < ns)
                place(i);
            else
                miss[i - ns] = !narrow(pieces[i - ns]);
        };
        if (big)
            HostPool::get().run(ns + np, task);
        else
            for (std::size_t i = 0; i < ns + np; ++i) task(i);
        bool fits = true, cols_ok = true;
        for (std::size_t i = 0; i < np; ++i)
            if (miss[i]) (pieces[i].kind == I8V ? fits : cols_ok) = false;
        t_place += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tp).count();
        return {fits, cols_ok};
    };
    auto [fits, cols_ok] = build_image(va_narrow ? 1 : 8);
    if (cols_ok && !fits) {  // a value outside int8: int64 values
        if (!img_borrowed_) client_image_give(ctx_, img_);
        std::tie(fits, cols_ok) = build_image(8);
    }
    if (!cols_ok) {  // the constructor throws: hand back what it holds, then raise in order
        if (!img_borrowed_) client_image_give(ctx_, img_);
        img_ = ClientImage{};
        if (hit) plan_cache_give(ctx_, std::move(lease_));
        lease_ = PlanLease{};
        for (const CsrView& m : ms) col_check(m);
        throw std::logic_error("spmv: column check disagreement");
    }
    if (trace) {
        const auto t2 = std::chrono::steady_clock::now();
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        std::fprintf(stderr, "e2e-trace append %.1f image %.1f (take %.1f place+narrow %.1f) us\n", us(ts, t1),
                     us(t1, t2), us(t1, t1b), t_place);
    }
    if (hit) return;
    lease_.key = std::move(key);
    lease_.a.assign(n, 0);
    lease_.b.assign(n, 0);
    lease_.out.assign(n_dout_, 0);
    try {
        check_status(spmvgpu_ct_alloc(ctx_, n, lease_.a.data()));
        check_status(spmvgpu_ct_alloc(ctx_, n, lease_.b.data()));
        check_status(spmvgpu_ct_alloc(ctx_, n_dout_, lease_.out.data()));
    } catch (...) {
        plan_lease_free(ctx_, lease_);
        if (!img_borrowed_) client_image_give(ctx_, img_);
        throw;
    }
}

// The shape half of csr_to_cssc + generate_chunks for rows [r0, r1) of m
// (sparse.cpp:79-117, chunk.cpp:10-52): a stable counting sort of the rows by
// descending length gives the CSSC row order; aligned column j has height
// h_j = #rows longer than j; chunks open at a column, fix h, and admit columns
// while h (k + 1) <= budget.  The entries themselves are scattered on the
// device (k_pack_cssc) from the row records built here.  Independent per
// slice (chunk indices and the slice id are local, fixed up when the records
// are placed into the client image).
void BatchedSpmv::shape_slice(const CsrView& m, const SliceJob& job, std::size_t budget, SliceShape& s) const {
    // per-slice checks in the reference's order (protocol.cpp:80-90)
    if (budget == 0 || budget > hp_.slot_count)
        throw std::invalid_argument("spmv: chunk_size must be in [1, slot_count]");
    s.mat = job.mat;
    s.rows = job.r1 - job.r0;
    s.vec_base = static_cast<std::int32_t>(job.vec_base);
    const std::uint64_t* rp = m.row_ptrs + job.r0;
    std::size_t max_len = 0;
    for (std::size_t i = 0; i < s.rows; ++i) max_len = std::max<std::size_t>(max_len, rp[i + 1] - rp[i]);
    // histogram of the lengths, slot max_len - len + 1 (descending order);
    // height[j] = #rows longer than j is its suffix sum
    std::vector<std::uint32_t> bucket(max_len + 2, 0);
    for (std::size_t i = 0; i < s.rows; ++i) ++bucket[max_len - (rp[i + 1] - rp[i]) + 1];
    std::vector<std::size_t> height(max_len, 0);
    for (std::size_t acc = 0, len = max_len; len >= 1; --len) {
        acc += bucket[max_len - len + 1];
        height[len - 1] = acc;
    }
    if (max_len && height[0] > budget)
        throw ColumnTooTallError("generate_chunks: aligned column 0 has height " + std::to_string(height[0]) +
                                 " > budget " + std::to_string(budget) + "; partition the rows first");
    std::partial_sum(bucket.begin(), bucket.end(), bucket.begin());
    // stable counting sort (the CSSC row order) and, in the same pass, the
    // device row records {nz_begin, len, pos, slice} of the non-empty rows,
    // which take the first height[0] positions
    const std::size_t nonempty = max_len ? height[0] : 0;
    s.rowrec.resize(4 * nonempty);
    std::int32_t* rr = s.rowrec.data();
    s.row_map.resize(s.rows);
    for (std::size_t i = 0; i < s.rows; ++i) {
        const std::size_t len = rp[i + 1] - rp[i];
        const std::uint32_t p = bucket[max_len - len]++;
        s.row_map[p] = i;
        if (len) {
            rr[4 * p] = static_cast<std::int32_t>(job.nz_base + static_cast<std::int64_t>(rp[i]));
            rr[4 * p + 1] = static_cast<std::int32_t>(len);
            rr[4 * p + 2] = static_cast<std::int32_t>(p);
            rr[4 * p + 3] = 0;  // slice id, set when placed
        }
    }
    s.colrec.resize(4 * max_len);
    std::int32_t* cr = s.colrec.data();
    std::size_t cw = 0;
    for (std::size_t first = 0; first < max_len;) {
        const std::size_t h = height[first];
        const std::size_t fit = std::min<std::size_t>(budget / h, max_len - first);
        const auto chunk = static_cast<std::int32_t>(s.r.size());  // local; offset when placed
        for (std::size_t k = 0; k < fit; ++k, cw += 4) {
            cr[cw] = chunk;
            cr[cw + 1] = static_cast<std::int32_t>(k);
            cr[cw + 2] = static_cast<std::int32_t>(h);
            cr[cw + 3] = 0;
        }
        s.r.push_back(h);
        s.c.push_back(fit);
        first += fit;
    }
}

void BatchedSpmv::append_slice(SliceShape& sh, std::size_t col_base) {
    Slice s;
    s.mat = sh.mat;
    s.rows = sh.rows;
    s.row_map = std::move(sh.row_map);
    s.first_chunk = r_.size();
    r_.insert(r_.end(), sh.r.begin(), sh.r.end());
    c_.insert(c_.end(), sh.c.begin(), sh.c.end());
    s.n_ct = r_.size() - s.first_chunk;
    slicerec_.insert(slicerec_.end(), {static_cast<std::int32_t>(col_base), sh.vec_base});
    if (s.n_ct) s.result = static_cast<int>(n_out_++);
    for (std::size_t i = 0; i < s.n_ct; ++i) slice_id_.push_back(static_cast<std::uint32_t>(s.result));
    slices_.push_back(std::move(s));
}

BatchedSpmv::~BatchedSpmv() {
    if (img_.p) {
        if (encrypted_ && !done_) spmvgpu_sync(ctx_);  // the upload may still read the image
        if (!img_borrowed_) client_image_give(ctx_, img_);
    }
    if (lease_.key.empty()) return;
    if (done_)
        plan_cache_give(ctx_, std::move(lease_));
    else  // an evaluation that did not complete: do not keep its buffers
        plan_lease_free(ctx_, lease_);
}

void BatchedSpmv::encrypt() {
    const cssc::NvtxRange nvtx_("cssc.encrypt");
    const std::size_t n = dr_.size();
    if (!n) return;
    std::vector<spmvgpu_ct> all(lease_.a);
    all.insert(all.end(), lease_.b.begin(), lease_.b.end());
    if (encrypted_) spmvgpu_sync(ctx_);  // re-encryption rewrites the image's stream ids
    client_image_encrypt(ctx_, img_, all.data());
    encrypted_ = true;
    h2d_ = img_.bytes;
}

void BatchedSpmv::ensure_plan() {
    const cssc::NvtxRange nvtx_("cssc.plan");
    if (lease_.plan || dr_.empty()) return;
    check_status(spmvgpu_plan_create(ctx_, dr_.size(), dr_.data(), dc_.data(), dslice_.data(), n_dout_,
                                     lease_.a.data(), lease_.b.data(), lease_.out.data(), &lease_.plan));
}

void BatchedSpmv::cloud(bool use_graph) {
    const cssc::NvtxRange nvtx_("cssc.cloud");
    if (dr_.empty()) return;
    ensure_plan();
    // a plan seen before is worth a graph: capture on its second use
    if ((use_graph || lease_.uses > 0) && !lease_.captured) {
        check_status(spmvgpu_plan_capture(lease_.plan));
        lease_.captured = true;
    }
    check_status(spmvgpu_plan_run(lease_.plan));
    ++lease_.uses;
}

std::vector<std::uint64_t> BatchedSpmv::result_words() {
    std::uint64_t n = 0, slots = 0, ctw = 0, kw = 0;
    int dnum = 0;
    check_status(spmvgpu_ctx_sizes(ctx_, &n, &slots, &ctw, &kw, &dnum));
    std::vector<std::uint64_t> w(n_out_ * ctw, 0);
    for (std::size_t r = 0; r < n_out_; ++r)
        if (res_local_[r] >= 0)
            check_status(spmvgpu_ct_download(ctx_, lease_.out[static_cast<std::size_t>(res_local_[r])],
                                             w.data() + r * ctw));
    if (!n_out_) check_status(spmvgpu_sync(ctx_));
    return w;
}

std::vector<SpmvResult> BatchedSpmv::finish() {
    const cssc::NvtxRange nvtx_("cssc.decrypt");
    if (world_ > 1)
        throw std::invalid_argument("finish: a sharded job holds partial results; sum result_words() across "
                                    "ranks and call finish_words()");
    std::vector<spmvgpu_ct> outs(n_out_);
    for (std::size_t r = 0; r < n_out_; ++r) outs[r] = lease_.out[static_cast<std::size_t>(res_local_[r])];
    return decrypt_and_report(outs);
}

std::vector<SpmvResult> BatchedSpmv::finish_words(const std::uint64_t* words) {
    std::uint64_t n = 0, slots = 0, ctw = 0, kw = 0;
    int dnum = 0;
    check_status(spmvgpu_ctx_sizes(ctx_, &n, &slots, &ctw, &kw, &dnum));
    std::vector<spmvgpu_ct> tmp(n_out_, 0);
    if (n_out_) check_status(spmvgpu_ct_alloc(ctx_, n_out_, tmp.data()));
    try {
        for (std::size_t r = 0; r < n_out_; ++r) check_status(spmvgpu_ct_upload(ctx_, tmp[r], words + r * ctw));
        auto res = decrypt_and_report(tmp);
        if (n_out_) spmvgpu_ct_free(ctx_, tmp.data(), tmp.size());
        return res;
    } catch (...) {
        if (n_out_) spmvgpu_ct_free(ctx_, tmp.data(), tmp.size());
        throw;
    }
}

void BatchedSpmv::result_words_dev(std::uint64_t* dev) {
    std::uint64_t n = 0, slots = 0, ctw = 0, kw = 0;
    int dnum = 0;
    check_status(spmvgpu_ctx_sizes(ctx_, &n, &slots, &ctw, &kw, &dnum));
    auto* st = static_cast<cudaStream_t>(spmvgpu_stream(ctx_));
    for (std::size_t r = 0; r < n_out_; ++r) {
        std::uint64_t* dst = dev + r * ctw;
        cudaError_t e;
        if (res_local_[r] >= 0)
            e = cudaMemcpyAsync(dst, reinterpret_cast<const void*>(lease_.out[static_cast<std::size_t>(res_local_[r])]),
                                8 * ctw, cudaMemcpyDeviceToDevice, st);
        else
            e = cudaMemsetAsync(dst, 0, 8 * ctw, st);
        if (e != cudaSuccess) throw std::runtime_error(std::string("result_words_dev: ") + cudaGetErrorString(e));
    }
    check_status(spmvgpu_sync(ctx_));  // the caller's collective runs on another stream
}

std::vector<SpmvResult> BatchedSpmv::finish_words_dev(std::uint64_t* dev) {
    std::uint64_t n = 0, slots = 0, ctw = 0, kw = 0;
    int dnum = 0;
    check_status(spmvgpu_ctx_sizes(ctx_, &n, &slots, &ctw, &kw, &dnum));
    check_status(spmvgpu_fold_mod(ctx_, dev, n_out_));
    std::vector<spmvgpu_ct> tmp(n_out_, 0);
    if (n_out_) check_status(spmvgpu_ct_alloc(ctx_, n_out_, tmp.data()));
    try {
        auto* st = static_cast<cudaStream_t>(spmvgpu_stream(ctx_));
        for (std::size_t r = 0; r < n_out_; ++r) {
            const cudaError_t e = cudaMemcpyAsync(reinterpret_cast<void*>(tmp[r]), dev + r * ctw, 8 * ctw,
                                                  cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) throw std::runtime_error(std::string("finish_words_dev: ") + cudaGetErrorString(e));
        }
        auto res = decrypt_and_report(tmp);
        if (n_out_) spmvgpu_ct_free(ctx_, tmp.data(), tmp.size());
        return res;
    } catch (...) {
        if (n_out_) spmvgpu_ct_free(ctx_, tmp.data(), tmp.size());
        throw;
    }
}

std::vector<SpmvResult> BatchedSpmv::run_all(std::int64_t* const* out_values) {
    const cssc::NvtxRange nvtx_("cssc.spmv_batch");
    // first use of a plan, sharded jobs: the staged calls; a plan seen before:
    // pack, encryption, cloud, decryption and download as one graph launch
    if (dr_.empty() || world_ > 1 || lease_.uses == 0) {
        encrypt();
        cloud(false);
        return finish();
    }
    static const bool trace = std::getenv("CSSC_TRACE_E2E") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    ensure_plan();
    if (!pipeline_ready(lease_, img_)) pipeline_prepare(ctx_, lease_, img_);
    if (img_.p != lease_.pimg) std::memcpy(lease_.pimg, img_.p, img_.bytes);
    std::vector<spmvgpu_ct> all(lease_.a);
    all.insert(all.end(), lease_.b.begin(), lease_.b.end());
    client_image_fill(ctx_, lease_.pimg, img_, all.data());
    encrypted_ = true;
    h2d_ = img_.bytes;
    const auto t1 = std::chrono::steady_clock::now();
    pipeline_run(ctx_, lease_);
    const auto t2 = std::chrono::steady_clock::now();
    ++lease_.uses;
    if (trace) {
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        std::fprintf(stderr, "e2e-trace prepare %.1f graph+sync %.1f us\n", us(t0, t1), us(t1, t2));
    }
    // the pinned download holds each result's slots [0, rows) as u32 (the rest
    // are zero): read in place, no S-slot copy per result
    std::vector<SlotSource> src(n_out_);
    std::vector<std::int32_t> measured(n_out_, 0);
    for (std::size_t r = 0; r < n_out_; ++r) {  // world == 1: every result is local
        const PipelineResult pr = pipeline_result(lease_, res_local_[r]);
        src[r] = SlotSource{nullptr, pr.slots, static_cast<std::size_t>(pr.rows)};
        const int bl = pr.maxdev ? 64 - __builtin_clzll(pr.maxdev) : 0;
        measured[r] = std::max(0, 63 - bl);
    }
    const auto t3 = std::chrono::steady_clock::now();
    auto res = report(src, measured, out_values);
    d2h_ = pipeline_out_bytes(lease_);
    if (trace) {
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        std::fprintf(stderr, "e2e-trace results %.1f report %.1f us\n", us(t2, t3),
                     us(t3, std::chrono::steady_clock::now()));
    }
    return res;
}

std::vector<SpmvResult> BatchedSpmv::decrypt_and_report(const std::vector<spmvgpu_ct>& outs) {
    const std::size_t S = hp_.slot_count;
    std::vector<std::uint64_t> slots(n_out_ * S);
    std::vector<std::int32_t> measured(n_out_, 0);
    if (n_out_)
        check_status(spmvgpu_decrypt(ctx_, outs.data(), n_out_, slots.data(), measured.data()));
    else
        check_status(spmvgpu_sync(ctx_));
    std::vector<SlotSource> src(n_out_);
    for (std::size_t r = 0; r < n_out_; ++r) src[r] = SlotSource{slots.data() + r * S, nullptr, S};
    auto res = report(src, measured);
    d2h_ = sizeof(std::uint64_t) * slots.size();
    return res;
}

std::vector<SpmvResult> BatchedSpmv::report(const std::vector<SlotSource>& slots,
                                            const std::vector<std::int32_t>& measured,
                                            std::int64_t* const* out_values) {
    const std::size_t S = hp_.slot_count;
    done_ = true;

    static const bool trace = std::getenv("CSSC_TRACE_E2E") != nullptr;
    double t_sched = 0, t_msgs = 0, t_noise = 0, t_rows = 0;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto dus = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    const auto tr0 = now();
    const NoiseModel& nm = hp_.noise;
    std::vector<SpmvResult> res(nmat_);
    struct Unpermute {  // one slice's decrypted rows -> original row order (rm, protocol.cpp:142-151)
        const Slice* s;
        std::int64_t* vals;
        const SlotSource* sl;
    };
    std::vector<Unpermute> unpermute;
    std::vector<std::size_t> row0(nmat_, 0);  // next row of each matrix
    for (std::size_t mi = 0; mi < nmat_; ++mi) {
        res[mi].message_ledger.key_holder = kh_;
        res[mi].noise_budget_remaining_bits = nm.initial_budget_bits;
        if (!out_values) res[mi].values.assign(rows_of_[mi], 0);
    }
    for (const Slice& s : slices_) {
        SpmvResult& R = res[s.mat];
        const std::size_t n_ct = s.n_ct;
        const std::uint64_t* rl = r_.data() + s.first_chunk;
        const std::uint64_t* cl = c_.data() + s.first_chunk;
        // ledger identities of one slice (protocol.cpp:99-136)
        OpLedger led;
        led.n_enc = 2 * n_ct;
        led.n_mult_cc = n_ct;
        led.n_mult_cp = n_ct;
        const auto ta = now();
        std::uint64_t rot = 0;
        std::vector<std::vector<RotStep>> sched(n_ct);
        for (std::size_t i = 0; i < n_ct; ++i) {
            sched[i] = rotation_schedule(rl[i], cl[i]);
            rot += sched[i].size();
        }
        led.n_rot = rot;
        led.n_add = rot + n_ct;
        led.n_dec = n_ct ? 1 : 0;
        R.op_ledger += led;
        R.n_ct += n_ct;
        const auto tb = now();
        t_sched += dus(ta, tb);
        // transcript (protocol.cpp:104-134)
        auto& msgs = R.message_ledger.messages;
        msgs.push_back({PartyRole::ClientA, PartyRole::Cloud, MessageKind::CiphertextBatch,
                        ciphertext_batch_bytes(hp_, n_ct), n_ct});
        msgs.push_back({PartyRole::ClientA, PartyRole::ClientB, MessageKind::ColumnIndexPlain,
                        column_index_bytes(rl, cl, n_ct), 0});
        msgs.push_back({PartyRole::ClientA, PartyRole::Cloud, MessageKind::ChunkShapeMeta,
                        4 + 8 * static_cast<std::uint64_t>(n_ct), 0});
        msgs.push_back({PartyRole::ClientB, PartyRole::Cloud, MessageKind::CiphertextBatch,
                        ciphertext_batch_bytes(hp_, n_ct), n_ct});
        const auto tc = now();
        t_msgs += dus(tb, tc);
        // model noise, replaying the backend's budget arithmetic
        int slice_noise = nm.initial_budget_bits;
        // this slice's rows (rows past the tallest chunk are 0)
        std::int64_t* vals = (out_values ? out_values[s.mat] : R.values.data()) + row0[s.mat];
        row0[s.mat] += s.rows;
        if (!n_ct && out_values) std::fill(vals, vals + s.rows, 0);
        if (n_ct) {
            msgs.push_back({PartyRole::Cloud, kh_, MessageKind::ResultCiphertext, ciphertext_batch_bytes(hp_, 1), 1});
            int res_b = nm.initial_budget_bits;
            for (std::size_t i = 0; i < n_ct; ++i) {
                const int prod_b = lowered(nm.initial_budget_bits, nm.cost_ct_ct_mult_bits);
                int acc_b = prod_b;
                for (const RotStep& st : sched[i]) {
                    const int rot_b = lowered(st.from_accumulator ? acc_b : prod_b, nm.cost_rot_bits);
                    acc_b = lowered(std::min(acc_b, rot_b), nm.cost_add_bits);
                }
                res_b = lowered(std::min(res_b, lowered(acc_b, nm.cost_ct_pt_mult_bits)), nm.cost_add_bits);
            }
            slice_noise = res_b;
            if (res_b <= 0)
                throw NoiseExhaustedError("decrypt: noise budget exhausted (slice result)");
            // the real BFV check: a result whose measured invariant-noise
            // budget is gone would decrypt to wrong values (he.cpp:84-91 semantics)
            const int meas = measured[static_cast<std::size_t>(s.result)];
            if (meas <= 0)
                throw NoiseExhaustedError("decrypt: measured invariant-noise budget exhausted (slice result)");
            const auto td = now();
            t_noise += dus(tc, td);
            unpermute.push_back({&s, vals, &slots[static_cast<std::size_t>(s.result)]});
            R.measured_noise_budget_bits =
                R.measured_noise_budget_bits < 0 ? meas : std::min(R.measured_noise_budget_bits, meas);
            t_noise += dus(td, now());
        }
        R.noise_budget_remaining_bits = std::min(R.noise_budget_remaining_bits, slice_noise);
    }
    const auto tu = now();
    const std::uint64_t t = hp_.plaintext_modulus, half = t / 2;  // to_signed: centred residue
    auto one = [&](std::size_t i) {
        const Unpermute& u = unpermute[i];
        const std::size_t avail = std::min({u.s->rows, S, u.sl->count});
        const std::size_t* rm = u.s->row_map.data();
        auto centred = [t, half](std::uint64_t r) {
            return static_cast<std::int64_t>(r) - (r > half ? static_cast<std::int64_t>(t) : 0);
        };
        if (u.sl->u64)
            for (std::size_t idx = 0; idx < avail; ++idx) u.vals[rm[idx]] = centred(u.sl->u64[idx]);
        else
            for (std::size_t idx = 0; idx < avail; ++idx) u.vals[rm[idx]] = centred(u.sl->u32[idx]);
        for (std::size_t idx = avail; idx < u.s->rows; ++idx) u.vals[rm[idx]] = 0;  // past the tallest chunk
    };
    std::size_t total_rows = 0;
    for (const auto& u : unpermute) total_rows += u.s->rows;
    if (total_rows >= (std::size_t{1} << 15) && unpermute.size() > 1)
        HostPool::get().run(unpermute.size(), one);
    else
        for (std::size_t i = 0; i < unpermute.size(); ++i) one(i);
    t_rows += dus(tu, now());
    if (trace)
        std::fprintf(stderr, "e2e-trace report: init+loop %.1f sched %.1f msgs %.1f noise %.1f rows %.1f us\n",
                     dus(tr0, now()), t_sched, t_msgs, t_noise, t_rows);
    return res;
}

}  // namespace spmv::detail
