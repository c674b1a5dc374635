// directory.cpp — see directory.hpp.
#include "directory.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>

#include "errc.hpp"

namespace trims {

namespace {
constexpr uint64_t kDirMagic = 0x31524944534d5254ull;  // "TRMSDIR1"
constexpr uint64_t kGold = 0x9e3779b97f4a7c15ull;

uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
}  // namespace

uint64_t fnv1a64(const std::string& s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001b3ull;
  }
  return h;
}

uint64_t peer_score(const std::string& key, int rank) { return mix(fnv1a64(key) ^ (uint64_t(rank) + 1) * kGold); }

struct Directory::Header {
  uint64_t magic;
  uint32_t world, slots;
  uint64_t reserved[6];
};
static_assert(sizeof(std::atomic<uint64_t>) == 8 && std::atomic<uint64_t>::is_always_lock_free);

struct alignas(64) Directory::Slot {
  std::atomic<uint64_t> seq;  // odd while the owning rank edits the slot
  uint32_t live, key_len;
  uint64_t key_hash;
  DirCoords c;
  char key[kKeyMax];
};

std::unique_ptr<Directory> Directory::open(const std::string& name, int world, int rank, uint32_t slots) {
  if (world < 1 || rank < 0 || rank >= world || slots == 0 || name.empty() || name.find('/') != std::string::npos)
    raise(Errc::InvalidArgument, "directory: bad name/world/rank/slots");
  std::unique_ptr<Directory> d(new Directory());
  d->world_ = world;
  d->rank_ = rank;
  d->slots_ = slots;
  d->bytes_ = sizeof(Header) + uint64_t(world) * slots * sizeof(Slot);
  const std::string path = "/" + name;
  d->fd_ = ::shm_open(path.c_str(), O_CREAT | O_RDWR | O_CLOEXEC, 0600);
  if (d->fd_ < 0) raise(Errc::Internal, "shm_open " + path + ": " + std::strerror(errno));
  struct stat st{};
  if (::fstat(d->fd_, &st) != 0) raise(Errc::Internal, "fstat " + path);
  // A fresh object reads as all-zero: every slot empty, no initialiser race.
  if (uint64_t(st.st_size) < d->bytes_ && ::ftruncate(d->fd_, off_t(d->bytes_)) != 0)
    raise(Errc::Internal, "ftruncate " + path + ": " + std::strerror(errno));
  d->map_ = ::mmap(nullptr, d->bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, d->fd_, 0);
  if (d->map_ == MAP_FAILED) {
    d->map_ = nullptr;
    raise(Errc::Internal, "mmap " + path);
  }
  auto* h = static_cast<Header*>(d->map_);
  if (h->magic == kDirMagic && (h->world != uint32_t(world) || h->slots != slots))
    raise(Errc::InvalidArgument, "directory " + path + " was created for world " + std::to_string(h->world) +
                                     " x " + std::to_string(h->slots) + " slots");
  h->world = uint32_t(world);  // every rank writes the same values
  h->slots = slots;
  std::atomic_ref<uint64_t>(h->magic).store(kDirMagic, std::memory_order_release);
  d->clear();
  return d;
}

void Directory::unlink(const std::string& name) { ::shm_unlink(("/" + name).c_str()); }

Directory::~Directory() {
  if (map_) {
    clear();
    ::munmap(map_, bytes_);
  }
  if (fd_ >= 0) ::close(fd_);
}

Directory::Slot* Directory::slot(int rank, uint32_t i) const {
  auto* base = reinterpret_cast<Slot*>(static_cast<char*>(map_) + sizeof(Header));
  return base + uint64_t(rank) * slots_ + i;
}

namespace {
template <class F>
void write_locked(std::atomic<uint64_t>& seq, F&& body) {
  const uint64_t s0 = seq.load(std::memory_order_relaxed);
  seq.store(s0 + 1, std::memory_order_relaxed);
  std::atomic_thread_fence(std::memory_order_release);
  body();
  seq.store(s0 + 2, std::memory_order_release);
}
}  // namespace

void Directory::publish(const fmt::ModelKey& key, const DirCoords& c) {
  const std::string k = fmt::to_string(key);
  if (k.size() >= kKeyMax) return;  // not directory-addressable; peers load it themselves
  const uint64_t kh = fnv1a64(k);
  Slot* target = nullptr;
  for (uint32_t i = 0; i < slots_ && !target; ++i) {
    Slot* s = slot(rank_, i);
    if (s->live && s->key_hash == kh && s->key_len == k.size() && std::memcmp(s->key, k.data(), k.size()) == 0)
      target = s;
  }
  for (uint32_t i = 0; i < slots_ && !target; ++i)
    if (!slot(rank_, i)->live) target = slot(rank_, i);
  if (!target) return;  // row full: the copy stays private to this rank
  DirCoords cc = c;
  cc.rank = rank_;
  write_locked(target->seq, [&] {
    target->live = 1;
    target->key_len = uint32_t(k.size());
    target->key_hash = kh;
    target->c = cc;
    std::memcpy(target->key, k.data(), k.size());
  });
}

void Directory::retract(const fmt::ModelKey& key) {
  const std::string k = fmt::to_string(key);
  const uint64_t kh = fnv1a64(k);
  for (uint32_t i = 0; i < slots_; ++i) {
    Slot* s = slot(rank_, i);
    if (s->live && s->key_hash == kh && s->key_len == k.size() && std::memcmp(s->key, k.data(), k.size()) == 0)
      write_locked(s->seq, [&] { s->live = 0; });
  }
}

void Directory::clear() {
  for (uint32_t i = 0; i < slots_; ++i) {
    Slot* s = slot(rank_, i);
    if (s->live) write_locked(s->seq, [&] { s->live = 0; });
  }
}

bool Directory::read_slot(const Slot& s, std::string* key, DirCoords* c) const {
  for (uint32_t spin = 0;; ++spin) {
    if (spin == (1u << 22)) return false;  // owner died mid-edit: treat the slot as empty
    const uint64_t s0 = s.seq.load(std::memory_order_acquire);
    if (s0 & 1) continue;  // the owner is mid-edit (a few stores long)
    const uint32_t live = s.live, klen = std::min<uint32_t>(s.key_len, kKeyMax);
    DirCoords cc;
    std::memcpy(&cc, &s.c, sizeof cc);
    char kb[kKeyMax];
    std::memcpy(kb, s.key, klen);
    std::atomic_thread_fence(std::memory_order_acquire);
    if (s.seq.load(std::memory_order_relaxed) != s0) continue;
    if (!live) return false;
    key->assign(kb, klen);
    *c = cc;
    return true;
  }
}

std::vector<DirCoords> Directory::holders(const fmt::ModelKey& key) const {
  const std::string k = fmt::to_string(key);
  std::vector<DirCoords> out;
  std::string sk;
  DirCoords c;
  for (int r = 0; r < world_; ++r) {
    if (r == rank_) continue;
    for (uint32_t i = 0; i < slots_; ++i)
      if (read_slot(*slot(r, i), &sk, &c) && sk == k) {
        out.push_back(c);
        break;
      }
  }
  std::sort(out.begin(), out.end(),
            [&](const DirCoords& a, const DirCoords& b) { return peer_score(k, a.rank) > peer_score(k, b.rank); });
  return out;
}

std::vector<std::pair<std::string, DirCoords>> Directory::row(int rank) const {
  if (rank < 0 || rank >= world_) raise(Errc::InvalidArgument, "directory: rank out of range");
  std::vector<std::pair<std::string, DirCoords>> out;
  std::string sk;
  DirCoords c;
  for (uint32_t i = 0; i < slots_; ++i)
    if (read_slot(*slot(rank, i), &sk, &c)) out.emplace_back(sk, c);
  return out;
}

bool peer_retryable(Errc e) {
  switch (e) {
    case Errc::StaleGeneration:
    case Errc::ChecksumMismatch:
    case Errc::NoSuchSegment:
    case Errc::NotSealed:
    case Errc::CudaError:
    case Errc::InvalidArgument:
    case Errc::Internal: return true;
    default: return false;
  }
}

PlacementResult open_with_peers(CacheCore& core, const Directory* dir, const fmt::ModelKey& key, const Granularity& g,
                                uint64_t now, const ManifestFn& manifest_for, const SourceFn& source_for,
                                PeerCounters* ctr, int* peer_rank) {
  if (peer_rank) *peer_rank = -1;
  if (dir && dir->world() > 1 && !core.fast_resident(key)) {
    std::vector<DirCoords> hs = dir->holders(key);
    std::shared_ptr<const fmt::Manifest> m = hs.empty() ? nullptr : manifest_for(key);
    for (const DirCoords& c : m ? hs : std::vector<DirCoords>{}) {
      if (ctr) ++ctr->attempts;
      std::shared_ptr<void> hold;
      try {
        PeerSource src = source_for(c, &hold);
        src.manifest = m;
        PlacementResult r = core.open_model(key, g, now, &src);
        if (peer_rank && r.outcome == Outcome::PeerHit) *peer_rank = c.rank;
        return r;
      } catch (const Error& e) {
        if (!peer_retryable(e.code())) {
          core.note_open_error();
          throw;
        }
        if (ctr) ++ctr->fallbacks;
      }
    }
  }
  return core.open_model(key, g, now);
}

}  // namespace trims
