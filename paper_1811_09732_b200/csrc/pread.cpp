// pread.cpp — see pread.hpp.
#include "pread.hpp"

#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <exception>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "errc.hpp"

namespace trims {

void pipelined_read(int fd, uint64_t off, uint64_t len, uint8_t* dst, unsigned threads, Sha256* hash,
                    const std::function<void(const uint8_t*, uint64_t, uint64_t)>& in_order) {
  const uint64_t pieces = (len + kReadPiece - 1) / kReadPiece;
  if (!pieces) return;
  const unsigned readers = unsigned(std::clamp<uint64_t>(pieces, 1, std::max(1u, threads)));
  // verify-only: a ring of slots, piece i in slot i % ring, reusable once
  // every consumer is past piece i - ring
  const uint64_t ring = dst ? pieces : std::min<uint64_t>(pieces, 2 * readers + 2);
  std::unique_ptr<uint8_t, void (*)(void*)> ring_mem(nullptr, std::free);
  if (!dst) {
    ring_mem.reset(static_cast<uint8_t*>(std::aligned_alloc(4096, ring * kReadPiece)));
    if (!ring_mem) raise(Errc::Internal, "read ring allocation failed");
  }
  auto at = [&](uint64_t i) { return dst ? dst + i * kReadPiece : ring_mem.get() + (i % ring) * kReadPiece; };
  const bool hashing = hash != nullptr, sinking = bool(in_order);

  std::mutex mu;
  std::condition_variable cv;
  std::vector<uint8_t> landed(pieces, 0);
  uint64_t next = 0, hashed = 0, sunk = 0;  // guarded by mu
  bool failed = false;
  std::exception_ptr err;
  auto retired = [&] {  // pieces every consumer is done with
    uint64_t r = pieces;
    if (hashing) r = std::min(r, hashed);
    if (sinking) r = std::min(r, sunk);
    return r;
  };
  auto fail = [&](std::exception_ptr e) {
    std::lock_guard lk(mu);
    if (!failed) err = e;
    failed = true;
    cv.notify_all();
  };

  auto reader = [&] {
    try {
      for (;;) {
        uint64_t i;
        {
          std::unique_lock lk(mu);
          if (failed || next >= pieces) return;
          i = next++;
          if (!dst) cv.wait(lk, [&] { return failed || i < retired() + ring; });
          if (failed) return;
        }
        const uint64_t b = i * kReadPiece, n = std::min(len - b, kReadPiece);
        uint8_t* p = at(i);
        for (uint64_t got = 0; got < n;) {
          ssize_t r = ::pread(fd, p + got, size_t(n - got), off_t(off + b + got));
          if (r <= 0) raise(Errc::Corrupt, "blob truncated (short read)");
          got += uint64_t(r);
        }
        std::lock_guard lk(mu);
        landed[i] = 1;
        cv.notify_all();
      }
    } catch (...) {
      fail(std::current_exception());
    }
  };
  // one in-order consumer: waits for piece i, runs fn, advances its cursor
  auto consume = [&](uint64_t& cursor, const std::function<void(const uint8_t*, uint64_t, uint64_t)>& fn) {
    for (uint64_t i = 0; i < pieces; ++i) {
      {
        std::unique_lock lk(mu);
        cv.wait(lk, [&] { return failed || landed[i]; });
        if (failed) return;
      }
      const uint64_t b = i * kReadPiece;
      fn(at(i), b, std::min(len - b, kReadPiece));
      std::lock_guard lk(mu);
      cursor = i + 1;
      cv.notify_all();
    }
  };

  std::vector<std::thread> ts;
  ts.reserve(readers + 1);
  for (unsigned r = 0; r < readers; ++r) ts.emplace_back(reader);
  if (hashing) {
    ts.emplace_back([&] {
      try {
        consume(hashed, [&](const uint8_t* p, uint64_t, uint64_t n) { hash->update(p, n); });
      } catch (...) {
        fail(std::current_exception());
      }
    });
  }
  if (sinking) {
    try {
      consume(sunk, in_order);
    } catch (...) {
      fail(std::current_exception());
    }
  }
  for (auto& t : ts) t.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace trims
