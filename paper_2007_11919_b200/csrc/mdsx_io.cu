// File ingestion for the drop-in dataio layer (reference dataio.py:42-130):
//   * IDX image / label headers validated like read_idx_images / read_idx_labels;
//   * IDX image payloads streamed straight into a device matrix: chunked reads
//     into two pinned buffers, the unsigned bytes cross PCIe (1/8 of the
//     float64 volume the reference materialises with .astype(float64)) and a
//     kernel widens them on the device, the read of chunk i+1 overlapping the
//     copy and kernel of chunk i;
//   * numeric CSV parsed by host threads (mmap, line index, per-thread ranges,
//     first error in file order), Python float() syntax, correctly rounded.
#include "mdsx_common.cuh"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

constexpr uint32_t IDX_IMAGES_MAGIC = 0x00000803u;
constexpr uint32_t IDX_LABELS_MAGIC = 0x00000801u;

int set_msg(char* msg, int64_t len, int code, const std::string& s) {
  if (msg && len > 0) {
    const size_t n = std::min<size_t>(s.size(), (size_t)len - 1);
    memcpy(msg, s.data(), n);
    msg[n] = 0;
  }
  return code;
}

uint32_t be32(const unsigned char* p) {
  return ((uint32_t)p[0] << 24) | ((uint32_t)p[1] << 16) | ((uint32_t)p[2] << 8) | (uint32_t)p[3];
}

std::string hex8(uint32_t v) {
  char b[16];
  snprintf(b, sizeof b, "0x%08x", v);
  return b;
}

// Header of an IDX file (dataio.py:42-58 images, 68-82 labels).  Returns the
// payload offset and element count via the out-params.
int idx_header(const char* path, int kind, int64_t* count, int32_t* height, int32_t* width,
               int64_t* payload_off, char* msg, int64_t msg_len) {
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return set_msg(msg, msg_len, MDSX_PARAM, std::string(path) + ": " + strerror(errno));
  struct stat sb;
  fstat(fd, &sb);
  const int64_t size = sb.st_size;
  const int hdr = kind == 3 ? 16 : 8;
  unsigned char h[16] = {0};
  const ssize_t got = size >= hdr ? pread(fd, h, hdr, 0) : 0;
  close(fd);
  const std::string what = kind == 3 ? "an IDX image header" : "an IDX label header";
  if (size < hdr || got != hdr)
    return set_msg(msg, msg_len, MDSX_FORMAT,
                   std::string(path) + ": file too short for " + what + " (" +
                       std::to_string(size) + " bytes)");
  const uint32_t magic = be32(h);
  const uint32_t want = kind == 3 ? IDX_IMAGES_MAGIC : IDX_LABELS_MAGIC;
  if (magic != want)
    return set_msg(msg, msg_len, MDSX_FORMAT,
                   std::string(path) + ": bad magic " + hex8(magic) + ", expected " + hex8(want) +
                       (kind == 3 ? " for images" : " for labels"));
  const int64_t n = be32(h + 4);
  const int64_t hh = kind == 3 ? be32(h + 8) : 1, ww = kind == 3 ? be32(h + 12) : 1;
  const int64_t expected = hdr + n * hh * ww;
  if (size != expected)
    return set_msg(msg, msg_len, MDSX_FORMAT,
                   std::string(path) + ": payload size mismatch, expected " +
                       std::to_string(expected) + " bytes, got " + std::to_string(size));
  *count = n;
  *height = (int32_t)hh;
  *width = (int32_t)ww;
  *payload_off = hdr;
  return MDSX_OK;
}

template <typename T>
__global__ void widen_u8_kernel(const unsigned char* __restrict__ src, T* __restrict__ dst,
                                int64_t n, double scale) {
  // 16 bytes per thread (one 128-bit load when the chunk is aligned)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 16;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; i < n; i += stride) {
    if (i + 16 <= n && ((reinterpret_cast<uintptr_t>(src + i) & 15) == 0)) {
      const uint4 v = *reinterpret_cast<const uint4*>(src + i);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          dst[i + 4 * q + b] = (T)(scale * (double)((w[q] >> (8 * b)) & 0xffu));
    } else {
      for (int64_t e = i; e < min(n, i + 16); ++e) dst[e] = (T)(scale * (double)src[e]);
    }
  }
}

// ---------------------------------------------------------------- CSV
// Python float() syntax (what dataio.py:120 calls): surrounding whitespace
// stripped, optional sign, decimal digits with single underscores between
// digits, optional fraction / exponent, or inf / infinity / nan (any case);
// no hexadecimal.  The conversion itself is glibc strtod (correctly rounded,
// like CPython's).
bool parse_py_float(const char* b, const char* e, double* out) {
  auto ws = [](char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f'; };
  while (b < e && ws(*b)) ++b;
  while (e > b && ws(e[-1])) --e;
  if (b == e) return false;
  char buf[128];
  std::string big;
  char* t = buf;
  const size_t n = (size_t)(e - b);
  if (n >= sizeof buf) {
    big.resize(n + 1);
    t = &big[0];
  }
  size_t k = 0;
  const char* s = b;
  if (*s == '+' || *s == '-') t[k++] = *s++;
  const char* body = s;
  // special values
  const size_t rem = (size_t)(e - body);
  auto ieq = [&](const char* w) {
    const size_t L = strlen(w);
    if (rem != L) return false;
    for (size_t i = 0; i < L; ++i)
      if ((body[i] | 0x20) != w[i]) return false;
    return true;
  };
  if (ieq("inf") || ieq("infinity") || ieq("nan")) {
    const double v = ieq("nan") ? NAN : INFINITY;
    *out = (b[0] == '-') ? -v : v;
    return true;
  }
  // digits [_digits]* [. digits [_digits]*] [e|E [sign] digits [_digits]*]
  bool any = false, prev_digit = false;
  bool seen_dot = false, seen_exp = false;
  for (; s < e; ++s) {
    const char c = *s;
    if (c >= '0' && c <= '9') {
      t[k++] = c;
      any = true;
      prev_digit = true;
    } else if (c == '_') {
      if (!prev_digit || s + 1 >= e || !(s[1] >= '0' && s[1] <= '9')) return false;
      prev_digit = false;
    } else if (c == '.' && !seen_dot && !seen_exp) {
      t[k++] = c;
      seen_dot = true;
      prev_digit = false;
    } else if ((c == 'e' || c == 'E') && !seen_exp && any) {
      t[k++] = c;
      seen_exp = true;
      prev_digit = false;
      if (s + 1 < e && (s[1] == '+' || s[1] == '-')) t[k++] = *++s;
      if (!(s + 1 < e && s[1] >= '0' && s[1] <= '9')) return false;
    } else {
      return false;
    }
  }
  if (!any) return false;
  t[k] = 0;
  char* endp = nullptr;
  const double v = strtod(t, &endp);
  if (endp != t + k) return false;
  *out = v;
  return true;
}

struct CsvFile {
  const char* data = nullptr;
  size_t size = 0;
  int fd = -1;
  std::vector<size_t> starts;   // record start offsets; record i ends at starts[i+1]-1 (the '\n')
  ~CsvFile() {
    if (data && size) munmap((void*)data, size);
    if (fd >= 0) close(fd);
  }
  int open_map(const char* path, char* msg, int64_t len) {
    fd = open(path, O_RDONLY);
    if (fd < 0) return set_msg(msg, len, MDSX_PARAM, std::string(path) + ": " + strerror(errno));
    struct stat sb;
    fstat(fd, &sb);
    size = (size_t)sb.st_size;
    if (size) {
      void* p = mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
      if (p == MAP_FAILED) return set_msg(msg, len, MDSX_PARAM, std::string(path) + ": mmap failed");
      data = (const char*)p;
      madvise(p, size, MADV_SEQUENTIAL);
    }
    for (size_t pos = 0; pos < size;) {
      starts.push_back(pos);
      const void* nl = memchr(data + pos, '\n', size - pos);
      pos = nl ? (size_t)((const char*)nl - data) + 1 : size;
    }
    starts.push_back(size);
    return MDSX_OK;
  }
  size_t records() const { return starts.size() - 1; }
  // [b, e) of record i without the line terminator ("\n" or "\r\n")
  void record(size_t i, const char*& b, const char*& e) const {
    b = data + starts[i];
    e = data + starts[i + 1];
    if (e > b && e[-1] == '\n') --e;
    if (e > b && e[-1] == '\r') --e;
  }
};

// Split one record into fields (csv module defaults: ',' delimiter, '"'
// quoting with doubled quotes).  An empty record has zero fields.
template <typename F>
int64_t split_fields(const char* b, const char* e, F&& on_field) {
  if (b == e) return 0;
  int64_t nf = 0;
  std::string q;
  const char* s = b;
  while (true) {
    if (s < e && *s == '"') {                  // quoted field
      q.clear();
      ++s;
      while (s < e) {
        if (*s == '"') {
          if (s + 1 < e && s[1] == '"') { q.push_back('"'); s += 2; continue; }
          ++s;
          break;
        }
        q.push_back(*s++);
      }
      while (s < e && *s != ',') q.push_back(*s++);   // text after the closing quote is kept
      on_field(nf, q.data(), q.data() + q.size());
    } else {
      const char* f = s;
      while (s < e && *s != ',') ++s;
      on_field(nf, f, s);
    }
    ++nf;
    if (s >= e) break;
    ++s;                                         // the delimiter
    if (s == e) { on_field(nf, s, s); ++nf; break; }   // trailing delimiter: one empty field
  }
  return nf;
}

}  // namespace

extern "C" {

int mdsx_idx_probe(const char* path, int32_t expect_kind, int64_t* count, int32_t* height,
                   int32_t* width, char* msg, int64_t msg_len) {
  if (expect_kind != 1 && expect_kind != 3)
    return set_msg(msg, msg_len, MDSX_PARAM, "expect_kind must be 1 (labels) or 3 (images)");
  int64_t off = 0;
  return idx_header(path, expect_kind, count, height, width, &off, msg, msg_len);
}

int mdsx_idx_load_images(mdsx_handle* h, const char* path, void* out, int dtype, double scale,
                         void* stream) {
  using namespace mdsx;
  if (!h) return MDSX_PARAM;
  if (dtype != MDSX_F64 && dtype != MDSX_F32) return fail(h, MDSX_PARAM, "dtype must be F64 or F32");
  char msg[512];
  int64_t count = 0, off = 0;
  int32_t hh = 0, ww = 0;
  int rc = idx_header(path, 3, &count, &hh, &ww, &off, msg, sizeof msg);
  if (rc) return fail(h, rc, msg);
  const int64_t total = count * (int64_t)hh * ww;
  if (total == 0) return MDSX_OK;
  cudaStream_t st = as_stream(stream);
  const int64_t CH = std::min<int64_t>(total, (int64_t)32 << 20);
  unsigned char* pin[2] = {nullptr, nullptr};
  unsigned char* dev[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  auto cleanup = [&]() {
    cudaStreamSynchronize(st);
    for (int b = 0; b < 2; ++b) {
      if (pin[b]) cudaFreeHost(pin[b]);
      if (dev[b]) cudaFree(dev[b]);
      if (done[b]) cudaEventDestroy(done[b]);
    }
  };
  for (int b = 0; b < 2; ++b) {
    if (cudaHostAlloc(&pin[b], CH, cudaHostAllocDefault) != cudaSuccess ||
        cudaMalloc(&dev[b], CH) != cudaSuccess ||
        cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming) != cudaSuccess) {
      cleanup();
      return fail(h, MDSX_CUDA, "idx staging allocation failed");
    }
  }
  const int fd = open(path, O_RDONLY);
  if (fd < 0) {
    cleanup();
    return fail(h, MDSX_PARAM, std::string(path) + ": " + strerror(errno));
  }
  posix_fadvise(fd, 0, 0, POSIX_FADV_SEQUENTIAL);
  const size_t es = dtype == MDSX_F64 ? 8 : 4;
  int64_t pos = 0;
  for (int c = 0; pos < total; ++c) {
    const int b = c & 1;
    const int64_t n = std::min(CH, total - pos);
    cudaEventSynchronize(done[b]);               // buffer b's previous copy has finished
    int64_t got = 0;
    while (got < n) {
      const ssize_t r = pread(fd, pin[b] + got, (size_t)(n - got), off + pos + got);
      if (r <= 0) {
        close(fd);
        cleanup();
        return fail(h, MDSX_FORMAT, std::string(path) + ": short read");
      }
      got += r;
    }
    cudaMemcpyAsync(dev[b], pin[b], (size_t)n, cudaMemcpyHostToDevice, st);
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((n + 16 * threads - 1) / (16 * threads), 8 * h->num_sms);
    pre(h, st);
    if (dtype == MDSX_F64)
      widen_u8_kernel<double><<<blocks, threads, 0, st>>>(dev[b], (double*)out + pos, n, scale);
    else
      widen_u8_kernel<float><<<blocks, threads, 0, st>>>(dev[b], (float*)out + pos, n, scale);
    if ((rc = launched(h, "widen_u8_kernel", st))) {
      close(fd);
      cleanup();
      return rc;
    }
    cudaEventRecord(done[b], st);
    pos += n;
  }
  close(fd);
  (void)es;
  cleanup();
  return cuda_check(h, cudaGetLastError(), "idx load");
}

int mdsx_csv_read(const char* path, int32_t has_header, int32_t threads, double* out,
                  int64_t* rows, int64_t* cols, char* msg, int64_t msg_len) {
  CsvFile f;
  int rc = f.open_map(path, msg, msg_len);
  if (rc) return rc;
  const size_t nrec = f.records();
  const size_t first = has_header ? 1 : 0;
  const int64_t nrows = nrec > first ? (int64_t)(nrec - first) : 0;
  int64_t width = 0;
  if (nrows > 0) {
    const char *b, *e;
    f.record(first, b, e);
    width = split_fields(b, e, [](int64_t, const char*, const char*) {});
  }
  if (!out) {                                   // sizing call
    *rows = nrows;
    *cols = width;
    return MDSX_OK;
  }
  if (*rows != nrows || *cols != width)
    return set_msg(msg, msg_len, MDSX_PARAM, "csv buffer shape does not match the sizing call");
  // parse: per-thread record ranges, first error (lowest line) wins
  int nt = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  nt = std::max(1, std::min<int>(nt, (int)std::max<int64_t>(1, nrows / 2048)));
  struct Err { int64_t line = INT64_MAX; std::string text; };
  std::vector<Err> errs(nt);
  auto work = [&](int t) {
    const int64_t r0 = nrows * t / nt, r1 = nrows * (t + 1) / nt;
    for (int64_t r = r0; r < r1; ++r) {
      const size_t rec = first + (size_t)r;
      const int64_t line_no = (int64_t)rec + 1;
      const char *b, *e;
      f.record(rec, b, e);
      double* row = out + r * width;
      int64_t bad_field = -1;
      std::string bad_text;
      const int64_t nf = split_fields(b, e, [&](int64_t j, const char* fb, const char* fe) {
        if (j >= width || bad_field >= 0) return;
        double v;
        if (parse_py_float(fb, fe, &v)) row[j] = v;
        else { bad_field = j; bad_text.assign(fb, fe); }
      });
      if (nf != width) {
        errs[t].line = line_no;
        errs[t].text = std::string(path) + ": ragged row at line " + std::to_string(line_no) +
                       ": expected " + std::to_string(width) + " fields, got " + std::to_string(nf);
        return;
      }
      if (bad_field >= 0) {
        errs[t].line = line_no;
        errs[t].text = std::string(path) + ": invalid number at line " + std::to_string(line_no) +
                       ": could not convert string to float: '" + bad_text + "'";
        return;
      }
    }
  };
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  const Err* best = nullptr;
  for (const Err& e : errs)
    if (e.line != INT64_MAX && (!best || e.line < best->line)) best = &e;
  if (best) return set_msg(msg, msg_len, MDSX_FORMAT, best->text);
  if (nrows == 0 || width == 0) return set_msg(msg, msg_len, MDSX_FORMAT, std::string(path) + ": no data rows");
  return MDSX_OK;
}

}  // extern "C"
