// pread.hpp — the disk side of the cold path: a file range read by several
// threads in 4 MiB pieces, with the pieces handed IN ORDER to a SHA-256 (on
// its own thread) and to a caller-side sink (the PCIe upload), so a verified
// load costs max(read, hash, upload) instead of their sum (
// replaces the reference's ifstream read + separate 1 MiB hash loop,
// model_format.cpp:370-429).
#pragma once

#include <cstdint>
#include <functional>

#include "sha256.hpp"

namespace trims {

constexpr uint64_t kReadPiece = 2ull << 20;  // measured: 2 MiB 4.3-4.4 ms vs 4 MiB 4.8 ms cold ResNet-50 (profiles/r01f/cold_read_ab.log)

// Reads [off, off+len) of fd in kReadPiece pieces (the last threads x
// kReadPiece bytes in half pieces; TRIMS_READ_PIECE_KB / _FINE_KB override).
// dst != nullptr: the bytes land there. dst == nullptr: pieces go through a
// small ring (verify-only). hash (optional) is updated with the range in order
// on a dedicated thread. sink (optional) is called on the calling thread once
// per piece after it has landed -- (piece pointer, byte offset within the
// range, bytes) -- in range order, or in landing order when sink_any_order
// (dst != nullptr only). A short read raises Corrupt; an exception from the
// sink stops the readers and is rethrown.
//
// direct_fd >= 0 (the same file opened O_DIRECT) with dst != nullptr: dst
// must be congruent to `off` modulo 4096 and the caller's allocation must
// span [dst - off % 4096, dst + len + 4096): the readers then read whole
// aligned 4 KiB blocks with O_DIRECT (DMA from the device into dst's pages,
// no page-cache copy; the bytes around the blob land in the slack). A piece
// the filesystem refuses (EINVAL) is read buffered instead. Hash and sink see
// exactly the blob range either way.
void pipelined_read(int fd, uint64_t off, uint64_t len, uint8_t* dst, unsigned threads, Sha256* hash,
                    const std::function<void(const uint8_t*, uint64_t, uint64_t)>& sink = {},
                    bool sink_any_order = false, int direct_fd = -1);

// Fraction of [off, off + len) of fd resident in the page cache (mincore over
// a sample of up to 256 pages); 1.0 when it cannot tell.
double page_cache_fraction(int fd, uint64_t off, uint64_t len);

}  // namespace trims
