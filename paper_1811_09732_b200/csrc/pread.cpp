// pread.cpp — see pread.hpp.
#include "pread.hpp"

#include <sys/mman.h>
#include <unistd.h>

#include <cerrno>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <exception>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "errc.hpp"

namespace trims {

namespace {

struct Piece {
  uint64_t begin, bytes;    // the blob range consumers see (offsets within [off, off + len))
  uint64_t rd_off, rd_len;  // what the reader reads: file offset, bytes
  int64_t rd_dst;           // ... to dst + rd_dst
};

uint64_t env_kb(const char* name, uint64_t dflt) {
  const char* e = std::getenv(name);
  return e ? std::max<uint64_t>(64, std::strtoull(e, nullptr, 10)) << 10 : dflt;
}

// kReadPiece pieces, except that the last `readers` x kReadPiece bytes are cut
// 2x finer: the final wave of reads then lands in small pieces, so the upload
// and hash left after the last read are short.
std::vector<Piece> cut(uint64_t len, unsigned readers) {
  static const uint64_t piece = env_kb("TRIMS_READ_PIECE_KB", kReadPiece);
  static const uint64_t fine = env_kb("TRIMS_READ_FINE_KB", kReadPiece / 2);
  std::vector<Piece> v;
  const uint64_t fine_from = len > uint64_t(readers) * piece ? len - uint64_t(readers) * piece : 0;
  for (uint64_t at = 0; at < len;) {
    const uint64_t step = at >= fine_from ? fine : piece;
    const uint64_t n = std::min(step, len - at);
    v.push_back({at, n, 0, n, int64_t(at)});
    at += n;
  }
  return v;
}

// Direct mode: cut the aligned superset [off - head, roundup(off + len)) of
// the blob into pieces (all multiples of 4 KiB), each mapped back onto the
// blob range its consumers see.
std::vector<Piece> cut_aligned(uint64_t off, uint64_t len, unsigned readers) {
  const uint64_t head = off % 4096, a0 = off - head;
  const uint64_t span = ((off + len + 4095) & ~4095ull) - a0;
  std::vector<Piece> v = cut(span, readers);  // 2 MiB / 1 MiB pieces: 4 KiB multiples
  std::vector<Piece> out;
  for (const Piece& p : v) {
    const uint64_t lo = std::max(p.begin, head), hi = std::min(p.begin + p.bytes, head + len);
    if (hi <= lo) continue;  // pure padding block (cannot happen: head < 4096 <= every piece)
    out.push_back({lo - head, hi - lo, a0 + p.begin, p.bytes, int64_t(p.begin) - int64_t(head)});
  }
  return out;
}

}  // namespace

double page_cache_fraction(int fd, uint64_t off, uint64_t len) {
  if (!len) return 1.0;
  const long pg = ::sysconf(_SC_PAGESIZE);
  const uint64_t a0 = off / pg * pg, span = off + len - a0;
  void* m = ::mmap(nullptr, size_t(span), PROT_READ, MAP_SHARED, fd, off_t(a0));
  if (m == MAP_FAILED) return 1.0;
  const uint64_t pages = (span + pg - 1) / pg;
  std::vector<unsigned char> vec(static_cast<size_t>(pages));
  double frac = 1.0;
  if (::mincore(m, size_t(span), vec.data()) == 0) {
    const uint64_t step = std::max<uint64_t>(1, pages / 256);
    uint64_t seen = 0, in = 0;
    for (uint64_t i = 0; i < pages; i += step, ++seen) in += vec[size_t(i)] & 1;
    frac = double(in) / double(seen);
  }
  ::munmap(m, size_t(span));
  return frac;
}

void pipelined_read(int fd, uint64_t off, uint64_t len, uint8_t* dst, unsigned threads, Sha256* hash,
                    const std::function<void(const uint8_t*, uint64_t, uint64_t)>& sink, bool sink_any_order,
                    int direct_fd) {
  if (!len) return;
  const unsigned want = std::max(1u, threads);
  const bool direct = direct_fd >= 0 && dst && (reinterpret_cast<uintptr_t>(dst) - off) % 4096 == 0;
  const std::vector<Piece> pieces = direct ? cut_aligned(off, len, want) : cut(len, want);
  const uint64_t np = pieces.size();
  const unsigned readers = unsigned(std::min<uint64_t>(np, want));
  if (!dst) sink_any_order = false;
  // verify-only: a ring of kReadPiece slots, piece i in slot i % ring,
  // reusable once every consumer is past piece i - ring
  const uint64_t ring = dst ? np : std::min<uint64_t>(np, 2 * readers + 2);
  uint64_t slot = 0;
  for (const Piece& p : pieces) slot = std::max<uint64_t>(slot, (p.bytes + 4095) & ~4095ull);
  std::unique_ptr<uint8_t, void (*)(void*)> ring_mem(nullptr, std::free);
  if (!dst) {
    ring_mem.reset(static_cast<uint8_t*>(std::aligned_alloc(4096, ring * slot)));
    if (!ring_mem) raise(Errc::Internal, "read ring allocation failed");
  }
  auto at = [&](uint64_t i) { return dst ? dst + pieces[i].begin : ring_mem.get() + (i % ring) * slot; };
  const bool hashing = hash != nullptr, sinking = bool(sink);

  std::mutex mu;
  std::condition_variable cv;
  std::vector<uint8_t> landed(np, 0), sunk_flag(np, 0);
  uint64_t next = 0, hashed = 0, sunk = 0;  // guarded by mu; sunk = pieces handed to the sink
  bool failed = false;
  std::exception_ptr err;
  auto retired = [&] {  // in-order prefix every consumer is done with (ring mode)
    uint64_t r = np;
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
          if (failed || next >= np) return;
          i = next++;
          if (!dst) cv.wait(lk, [&] { return failed || i < retired() + ring; });
          if (failed) return;
        }
        const Piece pc = pieces[i];
        if (direct) {
          // whole aligned blocks; the file may end inside the last one
          uint8_t* p = dst + pc.rd_dst;
          const uint64_t need = uint64_t(int64_t(pc.begin + pc.bytes) - pc.rd_dst);  // bytes up to the blob's end
          uint64_t got = 0;
          bool buffered = false;
          while (got < need) {
            ssize_t r = buffered ? ::pread(fd, p + got, size_t(need - got), off_t(pc.rd_off + got))
                                 : ::pread(direct_fd, p + got, size_t(pc.rd_len - got), off_t(pc.rd_off + got));
            if (r < 0 && !buffered && errno == EINVAL) {  // no O_DIRECT here: read this piece buffered
              buffered = true;
              continue;
            }
            if (r <= 0) raise(Errc::Corrupt, "blob truncated (short read)");
            got += uint64_t(r);
            if (!buffered && got % 4096) buffered = true;  // EOF inside a block: finish buffered
          }
        } else {
          uint8_t* p = at(i);
          for (uint64_t got = 0; got < pc.bytes;) {
            ssize_t r = ::pread(fd, p + got, size_t(pc.bytes - got), off_t(off + pc.begin + got));
            if (r <= 0) raise(Errc::Corrupt, "blob truncated (short read)");
            got += uint64_t(r);
          }
        }
        std::lock_guard lk(mu);
        landed[i] = 1;
        cv.notify_all();
      }
    } catch (...) {
      fail(std::current_exception());
    }
  };

  std::vector<std::thread> ts;
  ts.reserve(readers + 1);
  for (unsigned r = 0; r < readers; ++r) ts.emplace_back(reader);
  if (hashing) {
    ts.emplace_back([&] {
      try {
        for (uint64_t i = 0; i < np; ++i) {
          {
            std::unique_lock lk(mu);
            cv.wait(lk, [&] { return failed || landed[i]; });
            if (failed) return;
          }
          hash->update(at(i), pieces[i].bytes);
          std::lock_guard lk(mu);
          hashed = i + 1;
          cv.notify_all();
        }
      } catch (...) {
        fail(std::current_exception());
      }
    });
  }
  if (sinking) {
    try {
      uint64_t lo = 0;  // every piece below lo has been sunk
      for (uint64_t done = 0; done < np; ++done) {
        uint64_t i = np;
        {
          std::unique_lock lk(mu);
          cv.wait(lk, [&] {
            if (failed) return true;
            while (lo < np && sunk_flag[lo]) ++lo;
            if (!sink_any_order) return lo < np && landed[lo];
            for (uint64_t j = lo; j < next && j < np; ++j)
              if (landed[j] && !sunk_flag[j]) return true;
            return false;
          });
          if (failed) break;
          if (!sink_any_order) {
            i = lo;
          } else {
            for (uint64_t j = lo; j < np; ++j)
              if (landed[j] && !sunk_flag[j]) {
                i = j;
                break;
              }
          }
        }
        sink(at(i), pieces[i].begin, pieces[i].bytes);
        std::lock_guard lk(mu);
        sunk_flag[i] = 1;
        while (sunk < np && sunk_flag[sunk]) ++sunk;
        cv.notify_all();
      }
    } catch (...) {
      fail(std::current_exception());
    }
  }
  for (auto& t : ts) t.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace trims
