// cssc_io.cpp -- CSSC persistence.
//
// The reference persists a CSSC matrix only as the JSON that `spmv convert`
// writes (tools/spmv_main.cpp:39-58: csr_to_cssc, validate_cssc, then an
// ordered_json {rows, cols, va, ci, rm, cp} dumped with 2-space indent).
// cssc_to_json reproduces that text byte for byte (pinned against the
// reference built with nlohmann/json, tests/test_cssc_io.py); the binary form
// carries the same six fields compactly:
//   bytes 0-3   "CSSC"
//   byte  4     version (1)
//   byte  5     value width in bytes (1, 2, 4 or 8; two's complement)
//   byte  6     index width in bytes (4 or 8)
//   byte  7     0
//   8 x u64     rows, cols, nnz, aligned columns L
//   va[nnz], ci[nnz], rm[rows], cp[L + 1]  (little-endian, widths above)
// Loading checks every length and then validate_cssc; a malformed buffer
// raises ParseError (the reference's malformed-input exception).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>

#include "spmv/errors.hpp"
#include "spmv/sparse.hpp"

namespace spmv {

namespace {

constexpr std::size_t kHeader = 8 + 4 * 8;

int value_width(const std::vector<std::int64_t>& va) {
    std::int64_t lo = 0, hi = 0;
    for (std::int64_t v : va) {
        lo = std::min(lo, v);
        hi = std::max(hi, v);
    }
    if (lo >= INT8_MIN && hi <= INT8_MAX) return 1;
    if (lo >= INT16_MIN && hi <= INT16_MAX) return 2;
    if (lo >= INT32_MIN && hi <= INT32_MAX) return 4;
    return 8;
}

void put(std::vector<std::uint8_t>& out, std::uint64_t v, int width) {
    for (int b = 0; b < width; ++b) out.push_back(static_cast<std::uint8_t>(v >> (8 * b)));
}

std::uint64_t get(const std::uint8_t* p, int width) {
    std::uint64_t v = 0;
    for (int b = 0; b < width; ++b) v |= static_cast<std::uint64_t>(p[b]) << (8 * b);
    return v;
}

std::int64_t sign_extend(std::uint64_t v, int width) {
    if (width == 8) return static_cast<std::int64_t>(v);
    const int sh = 64 - 8 * width;
    return static_cast<std::int64_t>(v << sh) >> sh;
}

template <class V>
void json_array(std::string& s, const char* key, const V& a, bool last) {
    s += "  \"";
    s += key;
    s += "\": ";
    if (a.empty()) {
        s += "[]";
    } else {
        s += "[\n";
        for (std::size_t i = 0; i < a.size(); ++i) {
            s += "    ";
            s += std::to_string(a[i]);
            s += i + 1 < a.size() ? ",\n" : "\n";
        }
        s += "  ]";
    }
    s += last ? "\n" : ",\n";
}

}  // namespace

std::vector<std::uint8_t> cssc_to_bytes(const CsscMatrix& m) {
    const int vw = value_width(m.va);
    const std::uint64_t big = std::max<std::uint64_t>({m.rows, m.cols, m.nnz(), m.aligned_cols() + 1});
    const int iw = big >> 32 ? 8 : 4;
    std::vector<std::uint8_t> out;
    out.reserve(kHeader + m.nnz() * (vw + iw) + (m.rows + m.cp.size()) * iw);
    out.insert(out.end(), {'C', 'S', 'S', 'C', 1, static_cast<std::uint8_t>(vw), static_cast<std::uint8_t>(iw), 0});
    for (std::uint64_t v : {std::uint64_t{m.rows}, std::uint64_t{m.cols}, std::uint64_t{m.nnz()},
                            std::uint64_t{m.aligned_cols()}})
        put(out, v, 8);
    for (std::int64_t v : m.va) put(out, static_cast<std::uint64_t>(v), vw);
    for (std::size_t v : m.ci) put(out, v, iw);
    for (std::size_t v : m.rm) put(out, v, iw);
    if (m.cp.empty())
        put(out, 0, iw);  // L = 0: cp = {0}
    else
        for (std::size_t v : m.cp) put(out, v, iw);
    return out;
}

CsscMatrix cssc_from_bytes(std::span<const std::uint8_t> b) {
    if (b.size() < kHeader || std::memcmp(b.data(), "CSSC", 4) != 0 || b[4] != 1 || b[7] != 0)
        throw ParseError("cssc: not a CSSC v1 buffer", 0);
    const int vw = b[5], iw = b[6];
    if ((vw != 1 && vw != 2 && vw != 4 && vw != 8) || (iw != 4 && iw != 8))
        throw ParseError("cssc: bad field widths", 0);
    const std::uint64_t rows = get(b.data() + 8, 8), cols = get(b.data() + 16, 8), nnz = get(b.data() + 24, 8),
                        L = get(b.data() + 32, 8);
    if (rows > (std::uint64_t{1} << 40) || nnz > (std::uint64_t{1} << 40) || L > nnz)
        throw ParseError("cssc: implausible sizes", 0);
    const std::uint64_t need = kHeader + nnz * (vw + iw) + (rows + L + 1) * iw;
    if (b.size() != need) throw ParseError("cssc: length does not match the header", 0);
    CsscMatrix m;
    m.rows = rows;
    m.cols = cols;
    const std::uint8_t* p = b.data() + kHeader;
    m.va.resize(nnz);
    for (auto& v : m.va) v = sign_extend(get(p, vw), vw), p += vw;
    m.ci.resize(nnz);
    for (auto& v : m.ci) v = get(p, iw), p += iw;
    m.rm.resize(rows);
    for (auto& v : m.rm) v = get(p, iw), p += iw;
    m.cp.resize(L + 1);
    for (auto& v : m.cp) v = get(p, iw), p += iw;
    if (L == 0 && nnz == 0 && m.cp[0] == 0) m.cp.assign(1, 0);
    const auto bad = validate_cssc(m);
    if (!bad.empty()) throw ParseError("cssc: invalid structure: " + bad.front(), 0);
    return m;
}

std::string cssc_to_json(const CsscMatrix& m) {
    std::string s = "{\n";
    s += "  \"rows\": " + std::to_string(m.rows) + ",\n";
    s += "  \"cols\": " + std::to_string(m.cols) + ",\n";
    json_array(s, "va", m.va, false);
    json_array(s, "ci", m.ci, false);
    json_array(s, "rm", m.rm, false);
    json_array(s, "cp", m.cp, true);
    s += "}\n";
    return s;
}

}  // namespace spmv
