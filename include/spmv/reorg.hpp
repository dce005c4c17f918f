// spmv/reorg.hpp -- Client B's vector gather (reference reorg.hpp:14-21).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "spmv/chunk.hpp"

namespace spmv {

struct ReorgVector {
    std::vector<std::vector<std::int64_t>> segments;  // one per chunk, slot for slot
};

// IndexOutOfRangeError / DimensionMismatchError as the reference
ReorgVector reorg_vector(std::span<const std::int64_t> v, const ChunkSet& chunks);

}  // namespace spmv
