// Compiles the INTEGRATION.md shim against the reference headers and calls it
// (decode needs a GPU at run time).
#include <cstdio>
#include <vector>
#include "mvb_gpu.hpp"
int main() {
    const uint8_t fig1[] = {0x80, 0x01, 0x82, 0x03, 0x10, 0x20};
    std::vector<uint32_t> out(4);
    const mvb::DecodeResult r = mvb::gpu::decode_stream(fig1, 4, out.data());
    std::printf("status %d written %zu consumed %zu -> %u %u %u %u\n", static_cast<int>(r.status),
                r.values_written, r.bytes_consumed, out[0], out[1], out[2], out[3]);
    return (r.status == mvb::DecodeStatus::ok && out[1] == 386) ? 0 : 1;
}
