// stubs.cu — families not yet implemented report WL_EUNSUPPORTED.
#include "launch.h"
namespace wl {
namespace {
int unsup(const wl_block_desc& d) { return set_error(WL_EUNSUPPORTED, "block kind %d stride %d not implemented", d.kind, d.stride); }
int wc0(const wl_block_desc&) { return 0; }
int64_t wn0(const wl_block_desc&, int) { return 0; }
int64_t pb0(const wl_block_desc&) { return 0; }
int pk0(const wl_block_desc& d, const float* const*, uint8_t*) { return unsup(d); }
int64_t ws0(const wl_block_desc&) { return 0; }
int fw0(const wl_block_desc& d, const void*, const void*, void*, void*, cudaStream_t) { return unsup(d); }
}  // namespace
const Family kCf2Family = {unsup, wc0, wn0, pb0, pk0, ws0, fw0, nullptr};

const Family kStemFamily = {unsup, wc0, wn0, pb0, pk0, ws0, fw0, nullptr};
const Family kHeadFamily = {unsup, wc0, wn0, pb0, pk0, ws0, fw0, nullptr};
}  // namespace wl
