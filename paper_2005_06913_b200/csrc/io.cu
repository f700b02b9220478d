// Edge-list files: the reference's text format, parsed and
// written in parallel, and a binary SoA format that streams straight into
// HBM.
//
// Text: "<n> <m>\n" then m lines "<src> <dest> <weight>\n"
//   (/root/reference/proj/src/graph.cpp:228-295, load_graph / save_graph).
//   The loader keeps load_graph's strict rules and messages: header exactly
//   two integers, 1 <= n <= 2^32-1; exactly m edge lines of exactly three
//   integers (spaces between fields, a trailing '\r' tolerated); vertex ids
//   <= 2^32-1; only blank lines after the edge list. Any violation is
//   MST_ERR_PARSE (GraphError{ParseError}, graph.cpp:229-281). Weights must
//   fit 32 bits here (MST_ERR_WEIGHT), the device key's boundary narrowing.
//   The structural contract of build_graph (no self-loops / duplicates,
//   distinct weights, connectivity) is not enforced, as at the other entries.
//
// Binary SoA (".mstb"): a 4 KiB header, then the u32 src, dst and w arrays,
//   each starting on a 4 KiB boundary, so one sequential read per array
//   lands in a device buffer through two pinned staging chunks.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <omp.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace mstgpu {
void set_last_error(const std::string& m);

namespace {

constexpr char kMagic[8] = {'M', 'S', 'T', 'S', 'O', 'A', '0', '1'};
constexpr uint64_t kAlign = 4096;

struct BinHeader {
  char magic[8];
  uint32_t version;     // 1
  uint32_t weight_bits; // 32
  uint64_t n, m;
  uint64_t off_src, off_dst, off_w;  // byte offsets of the three arrays
};

uint64_t align_up(uint64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

[[noreturn]] void fail(int code, const std::string& msg) { throw MstError{code, msg}; }

template <class F>
int io_guarded(F&& f) {
  try {
    const int rc = f();
    if (rc == MST_OK) set_last_error("");
    return rc;
  } catch (const MstError& e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return MST_ERR_OOM;
  } catch (const std::exception& e) {
    set_last_error(std::string("internal error: ") + e.what());
    return MST_ERR_IO;
  }
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

// Read-only mapping of a whole file.
struct Mapped {
  const char* p = nullptr;
  size_t size = 0;
  Fd f;
  explicit Mapped(const std::string& path) {
    f.fd = open(path.c_str(), O_RDONLY);
    if (f.fd < 0) fail(MST_ERR_PARSE, "cannot open " + path);
    struct stat st;
    if (fstat(f.fd, &st) != 0) fail(MST_ERR_IO, "cannot stat " + path);
    size = (size_t)st.st_size;
    if (size) {
      void* m = mmap(nullptr, size, PROT_READ, MAP_PRIVATE | MAP_POPULATE, f.fd, 0);
      if (m == MAP_FAILED) fail(MST_ERR_IO, "cannot map " + path);
      p = static_cast<const char*>(m);
    }
  }
  ~Mapped() {
    if (p) munmap(const_cast<char*>(p), size);
  }
};

// load_graph's LineParser (graph.cpp:199-222): space-separated unsigned
// integers, nothing else on the line, one trailing '\r' tolerated.
struct LineParser {
  const char *p, *end;
  LineParser(const char* b, const char* e) : p(b), end(e) {
    if (p != end && end[-1] == '\r') --end;
  }
  bool next(uint64_t& out) {
    while (p != end && *p == ' ') ++p;
    if (p == end) return false;
    auto [ptr, ec] = std::from_chars(p, end, out);
    if (ec != std::errc{} || ptr == p) return false;
    p = ptr;
    return true;
  }
  bool at_end() {
    while (p != end && *p == ' ') ++p;
    return p == end;
  }
};

// Header line: [p, end of first line). Returns the body start.
const char* parse_header(const Mapped& f, const std::string& path, uint64_t& n, uint64_t& m) {
  if (f.size == 0) fail(MST_ERR_PARSE, path + ": empty file");
  const char* end = f.p + f.size;
  const char* nl = std::find(f.p, end, '\n');
  LineParser lp(f.p, nl);
  if (!lp.next(n) || !lp.next(m) || !lp.at_end()) fail(MST_ERR_PARSE, path + ": header must be \"<n> <m>\"");
  if (n < 1 || n > std::numeric_limits<uint32_t>::max())
    fail(MST_ERR_PARSE, path + ": bad vertex count " + std::to_string(n));
  return nl == end ? end : nl + 1;
}

void read_bin_header(int fd, const std::string& path, BinHeader& h) {
  if (pread(fd, &h, sizeof h, 0) != (ssize_t)sizeof h || std::memcmp(h.magic, kMagic, 8) != 0)
    fail(MST_ERR_PARSE, path + ": not an MSTSOA01 file");
  if (h.version != 1 || h.weight_bits != 32) fail(MST_ERR_PARSE, path + ": unsupported version");
  if (h.n < 1 || h.n > std::numeric_limits<uint32_t>::max()) fail(MST_ERR_PARSE, path + ": bad vertex count");
}

void pread_all(int fd, void* dst, size_t len, uint64_t off, const std::string& path) {
  // parallel page-cache copies: each thread reads a contiguous slice
  const int T = std::max(1, std::min(16, (int)(len >> 22)));
  bool bad = false;
#pragma omp parallel for num_threads(T) reduction(|| : bad)
  for (int t = 0; t < T; ++t) {
    const size_t lo = len * t / T, hi = len * (t + 1) / T;
    size_t done = lo;
    while (done < hi) {
      const ssize_t r = pread(fd, static_cast<char*>(dst) + done, hi - done, off + done);
      if (r <= 0) {
        bad = true;
        break;
      }
      done += (size_t)r;
    }
  }
  if (bad) fail(MST_ERR_IO, path + ": short read");
}

void pwrite_all(int fd, const void* src, size_t len, uint64_t off, const std::string& path) {
  size_t done = 0;
  while (done < len) {
    const ssize_t r = pwrite(fd, static_cast<const char*>(src) + done, len - done, off + done);
    if (r <= 0) fail(MST_ERR_IO, path + ": write failed");
    done += (size_t)r;
  }
}

struct Staging {
  static constexpr size_t kChunk = 32u << 20;
  std::mutex mu;
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaStream_t stream = nullptr;
};

Staging& staging_for(int dev) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<Staging>> pool;
  std::lock_guard<std::mutex> lock(mu);
  auto& slot = pool[dev];
  if (!slot) {
    auto s = std::make_unique<Staging>();
    MST_CUDA_CHECK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      MST_CUDA_CHECK(cudaHostAlloc(&s->buf[b], Staging::kChunk, cudaHostAllocDefault));
      MST_CUDA_CHECK(cudaEventCreateWithFlags(&s->ev[b], cudaEventDisableTiming));
    }
    slot = std::move(s);
  }
  return *slot;
}

}  // namespace
}  // namespace mstgpu

using namespace mstgpu;

extern "C" {

int mst_io_text_header(const char* path, uint32_t* out_n, uint64_t* out_m) {
  return io_guarded([&]() -> int {
    if (!path || !out_n || !out_m) fail(MST_ERR_INVALID_ARG, "NULL argument");
    // only the first line is needed: read a bounded prefix
    Fd f;
    f.fd = open(path, O_RDONLY);
    if (f.fd < 0) fail(MST_ERR_PARSE, std::string("cannot open ") + path);
    std::string head(256, '\0');
    const ssize_t r = pread(f.fd, head.data(), head.size(), 0);
    if (r <= 0) fail(MST_ERR_PARSE, std::string(path) + ": empty file");
    head.resize((size_t)r);
    const size_t nl = head.find('\n');
    LineParser lp(head.data(), head.data() + (nl == std::string::npos ? head.size() : nl));
    uint64_t n = 0, m = 0;
    if (!lp.next(n) || !lp.next(m) || !lp.at_end())
      fail(MST_ERR_PARSE, std::string(path) + ": header must be \"<n> <m>\"");
    if (n < 1 || n > std::numeric_limits<uint32_t>::max())
      fail(MST_ERR_PARSE, std::string(path) + ": bad vertex count " + std::to_string(n));
    *out_n = (uint32_t)n;
    *out_m = m;
    return MST_OK;
  });
}

int mst_io_load_text(const char* path, uint32_t n, uint64_t m, uint32_t* src, uint32_t* dst, uint32_t* w) {
  return io_guarded([&]() -> int {
    if (!path || (m && (!src || !dst || !w))) fail(MST_ERR_INVALID_ARG, "NULL argument");
    const std::string P(path);
    Mapped f(P);
    uint64_t hn = 0, hm = 0;
    const char* body = parse_header(f, P, hn, hm);
    if (hn != n || hm != m) fail(MST_ERR_INVALID_ARG, P + ": n/m differ from the header");
    const char* end = f.p + f.size;
    const size_t blen = (size_t)(end - body);
    // chunk the body at line starts; count lines per chunk, then parse each
    // chunk's lines into their global slots
    const int T = std::max(1, std::min(omp_get_max_threads(), (int)(blen >> 16) + 1));
    std::vector<const char*> cut(T + 1);
    cut[0] = body;
    cut[T] = end;
    for (int t = 1; t < T; ++t) {
      const char* c = body + blen * t / T;
      c = std::max(c, cut[t - 1]);
      const char* nl = std::find(c, end, '\n');
      cut[t] = nl == end ? end : nl + 1;
    }
    std::vector<uint64_t> lines(T + 1, 0);
#pragma omp parallel for num_threads(T)
    for (int t = 0; t < T; ++t) {
      const char *b = cut[t], *e = cut[t + 1];
      uint64_t c = (uint64_t)std::count(b, e, '\n');
      if (e > b && e[-1] != '\n') ++c;  // last line without a newline
      lines[t + 1] = c;
    }
    for (int t = 0; t < T; ++t) lines[t + 1] += lines[t];
    const uint64_t total_lines = lines[T];
    // first error in file order: (line index, code, message)
    std::vector<uint64_t> err_line(T, ~0ull);
    std::vector<int> err_code(T, 0);
    std::vector<std::string> err_msg(T);
#pragma omp parallel for num_threads(T)
    for (int t = 0; t < T; ++t) {
      const char* p = cut[t];
      const char* e = cut[t + 1];
      uint64_t i = lines[t];
      while (p < e) {
        const char* nl = std::find(p, e, '\n');
        LineParser lp(p, nl);
        if (i < m) {
          uint64_t s = 0, d = 0, wt = 0;
          if (!lp.next(s) || !lp.next(d) || !lp.next(wt) || !lp.at_end()) {
            err_line[t] = i;
            err_code[t] = MST_ERR_PARSE;
            err_msg[t] = P + ": edge line " + std::to_string(i + 1) + " must be \"<src> <dest> <weight>\"";
            break;
          }
          if (s > std::numeric_limits<uint32_t>::max() || d > std::numeric_limits<uint32_t>::max()) {
            err_line[t] = i;
            err_code[t] = MST_ERR_PARSE;
            err_msg[t] = P + ": vertex id overflow on line " + std::to_string(i + 2);
            break;
          }
          if (wt > std::numeric_limits<uint32_t>::max()) {
            err_line[t] = i;
            err_code[t] = MST_ERR_WEIGHT;
            err_msg[t] = P + ": weight on line " + std::to_string(i + 2) + " does not fit 32 bits";
            break;
          }
          src[i] = (uint32_t)s;
          dst[i] = (uint32_t)d;
          w[i] = (uint32_t)wt;
        } else if (!lp.at_end()) {
          err_line[t] = i;
          err_code[t] = MST_ERR_PARSE;
          err_msg[t] = P + ": trailing content after edge list";
          break;
        }
        ++i;
        p = nl == e ? e : nl + 1;
      }
    }
    int first = -1;
    for (int t = 0; t < T; ++t)
      if (err_line[t] != ~0ull && (first < 0 || err_line[t] < err_line[first])) first = t;
    // a short file is reported at the first missing line, after any earlier error
    if (total_lines < m && (first < 0 || err_line[first] >= total_lines))
      fail(MST_ERR_PARSE, P + ": expected " + std::to_string(m) + " edge lines, got " + std::to_string(total_lines));
    if (first >= 0) fail(err_code[first], err_msg[first]);
    return MST_OK;
  });
}

int mst_io_save_text(const char* path, uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                     const uint32_t* w) {
  return io_guarded([&]() -> int {
    if (!path || (m && (!src || !dst || !w))) fail(MST_ERR_INVALID_ARG, "NULL argument");
    const std::string P(path);
    // format in parallel chunks (save_graph's "%u %u %llu\n"), write in order
    const uint64_t kChunk = 1 << 20;
    const uint64_t nchunks = (m + kChunk - 1) / kChunk;
    Fd f;
    f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (f.fd < 0) fail(MST_ERR_IO, "save_graph: cannot open " + P);
    char head[64];
    const int hl = snprintf(head, sizeof head, "%llu %llu\n", (unsigned long long)n, (unsigned long long)m);
    uint64_t off = 0;
    pwrite_all(f.fd, head, (size_t)hl, off, P);
    off += (uint64_t)hl;
    const int T = std::max(1, std::min<int>(omp_get_max_threads(), 32));
    for (uint64_t c0 = 0; c0 < nchunks; c0 += (uint64_t)T) {
      const uint64_t cn = std::min<uint64_t>((uint64_t)T, nchunks - c0);
      std::vector<std::string> bufs(cn);
#pragma omp parallel for num_threads(T)
      for (int64_t k = 0; k < (int64_t)cn; ++k) {
        const uint64_t lo = (c0 + k) * kChunk, hi = std::min(m, lo + kChunk);
        std::string& b = bufs[k];
        b.resize((hi - lo) * 33);
        char* p = b.data();
        for (uint64_t i = lo; i < hi; ++i) {
          p = std::to_chars(p, p + 11, src[i]).ptr;
          *p++ = ' ';
          p = std::to_chars(p, p + 11, dst[i]).ptr;
          *p++ = ' ';
          p = std::to_chars(p, p + 11, w[i]).ptr;
          *p++ = '\n';
        }
        b.resize((size_t)(p - b.data()));
      }
      for (auto& b : bufs) {
        pwrite_all(f.fd, b.data(), b.size(), off, P);
        off += b.size();
      }
    }
    return MST_OK;
  });
}

int mst_io_save_soa(const char* path, uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                    const uint32_t* w) {
  return io_guarded([&]() -> int {
    if (!path || n < 1 || (m && (!src || !dst || !w))) fail(MST_ERR_INVALID_ARG, "bad argument");
    const std::string P(path);
    BinHeader h{};
    std::memcpy(h.magic, kMagic, 8);
    h.version = 1;
    h.weight_bits = 32;
    h.n = n;
    h.m = m;
    h.off_src = kAlign;
    h.off_dst = align_up(h.off_src + m * 4);
    h.off_w = align_up(h.off_dst + m * 4);
    Fd f;
    f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (f.fd < 0) fail(MST_ERR_IO, "cannot open " + P);
    std::vector<char> head(kAlign, 0);
    std::memcpy(head.data(), &h, sizeof h);
    pwrite_all(f.fd, head.data(), head.size(), 0, P);
    pwrite_all(f.fd, src, m * 4, h.off_src, P);
    pwrite_all(f.fd, dst, m * 4, h.off_dst, P);
    pwrite_all(f.fd, w, m * 4, h.off_w, P);
    if (ftruncate(f.fd, (off_t)(h.off_w + m * 4)) != 0) fail(MST_ERR_IO, P + ": truncate failed");
    return MST_OK;
  });
}

int mst_io_soa_header(const char* path, uint32_t* out_n, uint64_t* out_m) {
  return io_guarded([&]() -> int {
    if (!path || !out_n || !out_m) fail(MST_ERR_INVALID_ARG, "NULL argument");
    Fd f;
    f.fd = open(path, O_RDONLY);
    if (f.fd < 0) fail(MST_ERR_PARSE, std::string("cannot open ") + path);
    BinHeader h;
    read_bin_header(f.fd, path, h);
    *out_n = (uint32_t)h.n;
    *out_m = h.m;
    return MST_OK;
  });
}

int mst_io_load_soa(const char* path, uint32_t n, uint64_t m, uint32_t* src, uint32_t* dst, uint32_t* w,
                    int on_device) {
  return io_guarded([&]() -> int {
    if (!path || (m && (!src || !dst || !w))) fail(MST_ERR_INVALID_ARG, "NULL argument");
    const std::string P(path);
    Fd f;
    f.fd = open(path, O_RDONLY);
    if (f.fd < 0) fail(MST_ERR_PARSE, "cannot open " + P);
    BinHeader h;
    read_bin_header(f.fd, P, h);
    if (h.n != n || h.m != m) fail(MST_ERR_INVALID_ARG, P + ": n/m differ from the header");
    struct stat st;
    if (fstat(f.fd, &st) != 0 || (uint64_t)st.st_size < h.off_w + m * 4) fail(MST_ERR_PARSE, P + ": truncated");
    uint32_t* outs[3] = {src, dst, w};
    const uint64_t offs[3] = {h.off_src, h.off_dst, h.off_w};
    if (!on_device) {
      for (int a = 0; a < 3; ++a) pread_all(f.fd, outs[a], m * 4, offs[a], P);
      return MST_OK;
    }
    // file -> two pinned chunks -> HBM: the read of chunk k+1 overlaps the
    // copy of chunk k. The staging pair lives for the process (one per
    // device), so small files do not pay for pinned allocations.
    int dev = 0;
    MST_CUDA_CHECK(cudaGetDevice(&dev));
    Staging& sg = staging_for(dev);
    std::lock_guard<std::mutex> lock(sg.mu);
    bool busy[2] = {false, false};
    uint64_t k = 0;
    for (int a = 0; a < 3; ++a) {
      const uint64_t bytes = m * 4;
      for (uint64_t off = 0; off < bytes; off += Staging::kChunk, ++k) {
        const int b = (int)(k & 1);
        const size_t len = (size_t)std::min<uint64_t>(Staging::kChunk, bytes - off);
        if (busy[b]) MST_CUDA_CHECK(cudaEventSynchronize(sg.ev[b]));
        pread_all(f.fd, sg.buf[b], len, offs[a] + off, P);
        MST_CUDA_CHECK(cudaMemcpyAsync(reinterpret_cast<char*>(outs[a]) + off, sg.buf[b], len,
                                       cudaMemcpyHostToDevice, sg.stream));
        MST_CUDA_CHECK(cudaEventRecord(sg.ev[b], sg.stream));
        busy[b] = true;
      }
    }
    MST_CUDA_CHECK(cudaStreamSynchronize(sg.stream));
    return MST_OK;
  });
}

}  // extern "C"
