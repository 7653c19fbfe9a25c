// Host-side .bdelta container types (DeltaFile/DeltaEntry, P:include/deltakit/delta.hpp:76-93).
#pragma once

#include <stdint.h>

#include <string>
#include <vector>

namespace bd {

struct DeltaEntryHost {
    std::string name;
    bool packed = false;
    uint64_t rows = 0, cols = 0, planes = 0;
    std::vector<uint8_t> bits;   // planes * ceil(rows*cols/8)
    std::vector<float> scales;   // planes
    std::vector<float> raw;      // rows*cols (raw entries)
};

struct DeltaFileHost {
    std::vector<DeltaEntryHost> entries;
};

DeltaFileHost read_bdelta(const std::string& path);

}  // namespace bd
