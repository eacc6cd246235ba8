// mvb_gpu.hpp -- drop-in overloads with the reference's signatures.
#include <span>
#include <stdexcept>
#include "mvb/decode.hpp"   // reference types: DecodeResult, DecodeOptions, DecodeStatus
#include "mvb_cuda.h"       // this repository

namespace mvb::gpu {
inline DecodeResult to_ref(const mvb_result& r) {
    return {static_cast<DecodeStatus>(r.status), r.values_written, r.bytes_consumed};
}
// decode.hpp:44-45
inline DecodeResult decode_stream(std::span<const uint8_t> in, std::size_t count, uint32_t* out,
                                  const DecodeOptions& o = {}) {
    mvb_result r;
    const int rc = mvb_decode_stream(in.data(), in.size(), count, out,
                                     o.mode == DecodeMode::permissive ? MVB_PERMISSIVE : MVB_STRICT, &r);
    if (rc < 0) throw std::runtime_error("mvb_decode_stream failed");  // reference throws on misuse too
    return to_ref(r);
}
// decode.hpp:51-52
inline DecodeResult decode_delta_stream(std::span<const uint8_t> in, std::size_t count, uint32_t prev,
                                        uint32_t* out, const DecodeOptions& o = {}) {
    mvb_result r;
    const int rc = mvb_decode_delta_stream(in.data(), in.size(), count, prev, out,
                                           o.mode == DecodeMode::permissive ? MVB_PERMISSIVE : MVB_STRICT, &r);
    if (rc < 0) throw std::runtime_error("mvb_decode_delta_stream failed");
    return to_ref(r);
}
}  // namespace mvb::gpu
