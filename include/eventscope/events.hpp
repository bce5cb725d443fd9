// eventscope/events.hpp — event-model extract_features on the B200
// backend, from columnar events (TraceEvent numeric fields): validation,
// layer filter and the default per-layer features are computed on the device.
#pragma once

#include <cstdint>
#include <vector>

#include "eventscope/gmm.hpp"

namespace eventscope {

enum class Layer { Cuda = 0, Python = 1, Torch = 2, Nccl = 3, GpuSample = 4 };

struct EventColumns {                      // one entry per event; attrs NaN when absent
    std::vector<std::uint8_t> layer;       // Layer
    std::vector<std::int64_t> ts_start;    // ns, > 0
    std::vector<std::int64_t> duration_ns; // >= 0
    std::vector<double> message_bytes;     // Nccl (may be empty when there is no Nccl event)
    std::vector<double> util_pct, mem_used_mb, temp_c;  // GpuSample (may be empty likewise)
};

/// Cuda/Python/Torch: [log10(duration_ns + 1)]; Nccl: [log10(duration_ns + 1),
/// log10(message_bytes + 1)]; GpuSample: [util_pct, mem_used_mb, temp_c].  Rows keep event
/// order; event_index holds each row's source event.  Throws Data errors RangeViolation /
/// MissingField / UnknownLayer (first invalid event) and EmptyLayer.
FeatureMatrix extract_features(const EventColumns& events, Layer layer);

}  // namespace eventscope
