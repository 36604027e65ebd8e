// TT files (TTPAR1, core.py:364-398) straight to and from per-GPU slabs.
//
// File layout (save_tt, core.py:364-372): magic "TTPAR1", little-endian u64
// N, dims[N], ranks[N+1], then every core as raw little-endian f8 in F order
// (r_left, dim, r_right).  This rank's block of mode slices [lo, hi) of core
// n is r_right runs of r_left*(hi-lo) doubles, one per right-rank column,
// and those runs laid end to end are exactly the F-order device slab
// (r_left, hi-lo, r_right).  So a transfer is a stream of runs packed into
// page-locked staging buffers: while the host threads pread (pwrite) one
// buffer, the copy engine moves the other (double buffering on the context
// stream, one event per buffer).  Every rank reads / writes only its own
// runs: no gather to rank 0, no collective.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstring>
#include <thread>
#include <vector>

#include "ctx.cuh"

namespace ttb {

namespace {

constexpr size_t kStageBytes = size_t(64) << 20;  // per staging buffer
constexpr int kIoThreads = 8;

struct Piece {
  int64_t file_off;  // bytes
  size_t buf_off;    // bytes into the staging buffer
  size_t bytes;
};

// pread / pwrite a list of pieces with up to kIoThreads host threads
void host_io(int fd, bool write, char* buf, const std::vector<Piece>& pieces, const char* path) {
  size_t total = 0;
  for (const Piece& p : pieces) total += p.bytes;
  // split into roughly equal byte ranges over the pieces
  const int nt = (int)std::max<size_t>(1, std::min<size_t>(kIoThreads, total >> 22));
  std::vector<std::vector<Piece>> work(nt);
  const size_t share = (total + nt - 1) / nt;
  int t = 0;
  size_t acc = 0;
  for (Piece p : pieces) {
    while (p.bytes > 0) {
      const size_t room = share * (t + 1) > acc ? share * (t + 1) - acc : 0;
      const size_t take = (t == nt - 1) ? p.bytes : std::min(p.bytes, std::max<size_t>(room, 1));
      work[t].push_back({p.file_off, p.buf_off, take});
      p.file_off += (int64_t)take;
      p.buf_off += take;
      p.bytes -= take;
      acc += take;
      if (t < nt - 1 && acc >= share * (t + 1)) ++t;
    }
  }
  std::vector<int> err(nt, 0);
  auto run = [&](int k) {
    for (const Piece& p : work[k]) {
      size_t done = 0;
      while (done < p.bytes) {
        const ssize_t r = write ? pwrite(fd, buf + p.buf_off + done, p.bytes - done, p.file_off + (int64_t)done)
                                : pread(fd, buf + p.buf_off + done, p.bytes - done, p.file_off + (int64_t)done);
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) {
          err[k] = r == 0 ? -1 : errno;
          return;
        }
        done += (size_t)r;
      }
    }
  };
  std::vector<std::thread> th;
  for (int k = 1; k < nt; ++k) th.emplace_back(run, k);
  run(0);
  for (auto& x : th) x.join();
  for (int k = 0; k < nt; ++k) {
    if (err[k] == -1) TTB_THROW(TTB_ERR_SHAPE, std::string("TT file ") + path + " truncated");
    if (err[k]) TTB_THROW(TTB_ERR_CAPACITY, std::string(write ? "pwrite " : "pread ") + path + ": " + strerror(err[k]));
  }
}

struct Run {
  int64_t file_off;  // bytes
  double* dev;       // destination / source in device memory
  size_t bytes;
};

std::vector<Run> slab_runs(int64_t data_offset, int ndim, const int64_t* dims, const int64_t* ranks, const int64_t* lo,
                           const int64_t* hi, double* const* dev) {
  std::vector<Run> runs;
  int64_t base = data_offset;
  for (int n = 0; n < ndim; ++n) {
    const int64_t rl = ranks[n], I = dims[n], rr = ranks[n + 1];
    TTB_CHECK(rl >= 1 && rr >= 1 && I >= 1, TTB_ERR_SHAPE, "TT file: bad core shape");
    TTB_CHECK(0 <= lo[n] && lo[n] <= hi[n] && hi[n] <= I, TTB_ERR_SHAPE, "TT file: slice block out of range");
    const int64_t L = rl * (hi[n] - lo[n]);
    if (L > 0) {
      if (lo[n] == 0 && hi[n] == I) {
        runs.push_back({base, dev[n], (size_t)(8 * L * rr)});
      } else {
        for (int64_t c = 0; c < rr; ++c) runs.push_back({base + 8 * (rl * lo[n] + rl * I * c), dev[n] + L * c, (size_t)(8 * L)});
      }
    }
    base += 8 * rl * I * rr;
  }
  return runs;
}

// Walk the runs in staging-buffer sized groups.  Device destinations of
// consecutive runs within one slab are contiguous, so each group is a list
// of (device range) copies -- merged whenever contiguous.
struct Group {
  std::vector<Piece> pieces;
  std::vector<std::pair<double*, std::pair<size_t, size_t>>> copies;  // dev, (buf_off, bytes)
};

std::vector<Group> make_groups(const std::vector<Run>& runs) {
  std::vector<Group> groups(1);
  size_t fill = 0;
  for (Run r : runs) {
    while (r.bytes > 0) {
      if (fill == kStageBytes) {
        groups.emplace_back();
        fill = 0;
      }
      const size_t take = std::min(r.bytes, kStageBytes - fill);
      Group& g = groups.back();
      g.pieces.push_back({r.file_off, fill, take});
      if (!g.copies.empty()) {
        auto& last = g.copies.back();
        if ((char*)last.first + last.second.second == (char*)r.dev && last.second.first + last.second.second == fill) {
          last.second.second += take;
          goto next;
        }
      }
      g.copies.push_back({r.dev, {fill, take}});
    next:
      fill += take;
      r.file_off += (int64_t)take;
      r.dev = (double*)((char*)r.dev + take);
      r.bytes -= take;
    }
  }
  if (groups.back().pieces.empty()) groups.pop_back();
  return groups;
}

struct Staging {
  char* h[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~Staging() {
    for (int k = 0; k < 2; ++k) {
      if (h[k]) cudaFreeHost(h[k]);
      if (ev[k]) cudaEventDestroy(ev[k]);
    }
  }
};

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

void transfer(Ctx& ctx, const char* path, bool write, int64_t data_offset, int ndim, const int64_t* dims,
              const int64_t* ranks, const int64_t* lo, const int64_t* hi, double* const* dev) {
  TTB_CHECK(path && ndim >= 1, TTB_ERR_CONTRACT, "TT file: bad arguments");
  Fd f;
  f.fd = open(path, write ? O_WRONLY : O_RDONLY);
  TTB_CHECK(f.fd >= 0, TTB_ERR_SHAPE, std::string("cannot open TT file ") + path + ": " + strerror(errno));
  const std::vector<Group> groups = make_groups(slab_runs(data_offset, ndim, dims, ranks, lo, hi, dev));
  if (groups.empty()) return;
  if (!write) {
    struct stat st;
    TTB_CHECK(fstat(f.fd, &st) == 0, TTB_ERR_CAPACITY, std::string("fstat ") + path);
    int64_t end = data_offset;
    for (int n = 0; n < ndim; ++n) end += 8 * ranks[n] * dims[n] * ranks[n + 1];
    TTB_CHECK(st.st_size >= end, TTB_ERR_SHAPE, std::string("TT file ") + path + " truncated");
  }
  Staging s;
  for (int k = 0; k < 2; ++k) {
    TTB_CUDA(cudaHostAlloc((void**)&s.h[k], kStageBytes, cudaHostAllocDefault));
    TTB_CUDA(cudaEventCreateWithFlags(&s.ev[k], cudaEventDisableTiming));
  }
  if (!write) {
    // host fills buffer g%2 while the copy engine drains the other
    for (size_t g = 0; g < groups.size(); ++g) {
      const int k = (int)(g & 1);
      if (g >= 2) TTB_CUDA(cudaEventSynchronize(s.ev[k]));
      host_io(f.fd, false, s.h[k], groups[g].pieces, path);
      for (const auto& c : groups[g].copies)
        TTB_CUDA(cudaMemcpyAsync(c.first, s.h[k] + c.second.first, c.second.second, cudaMemcpyHostToDevice, ctx.stream));
      TTB_CUDA(cudaEventRecord(s.ev[k], ctx.stream));
    }
    TTB_CUDA(cudaStreamSynchronize(ctx.stream));
  } else {
    // device -> buffer g%2 is queued one group ahead of the host's pwrite
    auto enqueue = [&](size_t g) {
      const int k = (int)(g & 1);
      for (const auto& c : groups[g].copies)
        TTB_CUDA(cudaMemcpyAsync(s.h[k] + c.second.first, c.first, c.second.second, cudaMemcpyDeviceToHost, ctx.stream));
      TTB_CUDA(cudaEventRecord(s.ev[k], ctx.stream));
    };
    enqueue(0);
    for (size_t g = 0; g < groups.size(); ++g) {
      const int k = (int)(g & 1);
      TTB_CUDA(cudaEventSynchronize(s.ev[k]));
      if (g + 1 < groups.size()) enqueue(g + 1);
      host_io(f.fd, true, s.h[k], groups[g].pieces, path);
    }
  }
}

}  // namespace

}  // namespace ttb

using namespace ttb;

extern "C" {

int ttb_read_slabs(ttb_ctx* ctx, const char* path, int64_t data_offset, int ndim, const int64_t* dims,
                   const int64_t* ranks, const int64_t* lo, const int64_t* hi, double* const* out) {
  TTB_TRY_BEGIN
  TTB_CHECK(ctx, TTB_ERR_CONTRACT, "null context");
  transfer(ctx->c, path, false, data_offset, ndim, dims, ranks, lo, hi, out);
  TTB_TRY_END
}

int ttb_write_slabs(ttb_ctx* ctx, const char* path, int64_t data_offset, int ndim, const int64_t* dims,
                    const int64_t* ranks, const int64_t* lo, const int64_t* hi, const double* const* in) {
  TTB_TRY_BEGIN
  TTB_CHECK(ctx, TTB_ERR_CONTRACT, "null context");
  transfer(ctx->c, path, true, data_offset, ndim, dims, ranks, lo, hi, const_cast<double* const*>(in));
  TTB_TRY_END
}

}  // extern "C"
