// lorenz_io.cu — envelope format and the streaming file path (NEXT-2), host side of liblorenz.so.
//
// Files larger than HBM stream through the GPU in block-aligned chunks with four chunks in
// flight: while the host thread reads chunk i from disk into a pinned buffer, the GPU copies
// and encrypts chunks i-1..i-3 on their own streams and the finished chunk i-4 is written
// out. Only the public C ABI of lorenz.cu is used for the cipher itself.
//
// Envelope: "LZX1" | version 1 | mode | flags | dt_code | n_it u32 LE |
// chunk_size u32 LE (= B, 0 in STRONG) | payload_len u64 LE | ciphertext.
#include <cuda_runtime.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>

#include "../../include/lorenz.h"

namespace lz {
void set_last_error(const std::string& s);  // lorenz.cu
}

namespace {

// 4 chunks in flight of 32 MiB (measured best of 32/64/128 MiB on a 1 GiB file in tmpfs):
// pinning costs ~1 s per GB per call, so the staging (2 x 4 x 32 MiB) is kept small; the
// chunks' kernels overlap, so ~4 x 32768 lanes are in flight.
constexpr int kSlots = 4;
constexpr uint64_t kDefaultChunk = 32ull << 20;

void put_le(uint8_t* p, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
uint64_t get_le(const uint8_t* p, int n) {
  uint64_t v = 0;
  for (int i = n - 1; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

bool ok(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return true;
  lz::set_last_error(std::string(what) + ": " + cudaGetErrorString(e));
  return false;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// One streaming pass: blocks of the message move from `in` to `out` through the GPU.
// The calling thread reads chunk c into slot c % kSlots and enqueues H2D -> kernel -> D2H on
// the slot's stream; a writer thread waits for each slot's completion event in order, writes
// its output and frees the slot. Reads, GPU work and writes overlap.
struct Pipe {
  cudaStream_t st[kSlots] = {};
  cudaEvent_t done[kSlots] = {};
  uint8_t* h_in[kSlots] = {};
  uint8_t* h_out[kSlots] = {};
  uint8_t* d_in[kSlots] = {};
  uint8_t* d_out[kSlots] = {};
  lorenz_result* d_res = nullptr;
  // writer state
  std::mutex m;
  std::condition_variable cv;
  bool slot_free[kSlots];
  std::deque<std::pair<int, uint64_t>> wq;
  bool stop = false, started = false;
  lorenz_status werr = LORENZ_OK;
  FILE* out = nullptr;
  std::thread writer;
  double t_write = 0, t_wait_gpu = 0;

  lorenz_status init(uint64_t in_cap, uint64_t out_cap, FILE* o) {
    out = o;
    for (int s = 0; s < kSlots; ++s) {
      slot_free[s] = true;
      if (!ok(cudaStreamCreateWithFlags(&st[s], cudaStreamNonBlocking), "stream") ||
          !ok(cudaEventCreateWithFlags(&done[s], cudaEventDisableTiming), "event") ||
          !ok(cudaMallocHost(reinterpret_cast<void**>(&h_in[s]), in_cap ? in_cap : 16), "pinned in") ||
          !ok(cudaMallocHost(reinterpret_cast<void**>(&h_out[s]), out_cap ? out_cap : 16), "pinned out") ||
          !ok(cudaMalloc(reinterpret_cast<void**>(&d_in[s]), in_cap ? in_cap : 16), "device in") ||
          !ok(cudaMalloc(reinterpret_cast<void**>(&d_out[s]), out_cap ? out_cap : 16), "device out"))
        return LORENZ_E_CUDA;
    }
    if (!ok(cudaMalloc(reinterpret_cast<void**>(&d_res), sizeof(lorenz_result)), "result")) return LORENZ_E_CUDA;
    lorenz_status r = lorenz_result_init_async(d_res, st[0]);
    if (r != LORENZ_OK) return r;
    if (!ok(cudaStreamSynchronize(st[0]), "sync")) return LORENZ_E_CUDA;
    int dev = 0;
    cudaGetDevice(&dev);
    writer = std::thread([this, dev] { writer_loop(dev); });
    started = true;
    return LORENZ_OK;
  }
  void writer_loop(int dev) {
    cudaSetDevice(dev);
    for (;;) {
      std::pair<int, uint64_t> job;
      {
        std::unique_lock<std::mutex> lk(m);
        cv.wait(lk, [&] { return !wq.empty() || stop; });
        if (wq.empty()) return;
        job = wq.front();
        wq.pop_front();
      }
      const double t0 = now_s();
      lorenz_status s = LORENZ_OK;
      if (cudaEventSynchronize(done[job.first]) != cudaSuccess) s = LORENZ_E_CUDA;
      const double t1 = now_s();
      if (s == LORENZ_OK && job.second && fwrite(h_out[job.first], 1, job.second, out) != job.second)
        s = LORENZ_E_IO;
      const double t2 = now_s();
      {
        std::lock_guard<std::mutex> lk(m);
        t_wait_gpu += t1 - t0;
        t_write += t2 - t1;
        if (s != LORENZ_OK && werr == LORENZ_OK) werr = s;
        slot_free[job.first] = true;
      }
      cv.notify_all();
    }
  }
  // block until slot s is free (or the writer failed)
  lorenz_status acquire(int s) {
    std::unique_lock<std::mutex> lk(m);
    cv.wait(lk, [&] { return slot_free[s] || werr != LORENZ_OK; });
    return werr;
  }
  lorenz_status submit(int s, uint64_t outb) {
    if (!ok(cudaEventRecord(done[s], st[s]), "event record")) return LORENZ_E_CUDA;
    {
      std::lock_guard<std::mutex> lk(m);
      slot_free[s] = false;
      wq.emplace_back(s, outb);
    }
    cv.notify_all();
    return LORENZ_OK;
  }
  lorenz_status finish() {
    if (started) {
      {
        std::lock_guard<std::mutex> lk(m);
        stop = true;
      }
      cv.notify_all();
      writer.join();
      started = false;
    }
    return werr;
  }
  ~Pipe() {
    finish();
    for (int s = 0; s < kSlots; ++s) {
      if (st[s]) cudaStreamSynchronize(st[s]);
      if (done[s]) cudaEventDestroy(done[s]);
      if (h_in[s]) cudaFreeHost(h_in[s]);
      if (h_out[s]) cudaFreeHost(h_out[s]);
      if (d_in[s]) cudaFree(d_in[s]);
      if (d_out[s]) cudaFree(d_out[s]);
      if (st[s]) cudaStreamDestroy(st[s]);
    }
    if (d_res) cudaFree(d_res);
  }
};

struct File {
  FILE* f = nullptr;
  ~File() { if (f) fclose(f); }
};

lorenz_status stream_pass(const lorenz_key* k, uint64_t n, bool decrypt, FILE* in, FILE* out, uint64_t chunk_bytes,
                          lorenz_result* h_res) {
  lorenz_params p;
  if (lorenz_key_params(k, &p) != LORENZ_OK) return LORENZ_E_ARG;
  const uint64_t nb = lorenz_num_blocks(k, n);
  const bool fast = p.mode == LORENZ_FAST;
  const uint64_t B = fast ? p.block_size : n;
  uint64_t cb = fast ? (chunk_bytes ? chunk_bytes : kDefaultChunk) / p.block_size : 1;
  if (cb == 0) cb = 1;
  if (cb > nb) cb = nb;
  const uint64_t pt_cap = fast ? cb * B : n, ct_cap = pt_cap + 16 * cb;
  static const bool trace = std::getenv("LORENZ_IO_TRACE") != nullptr;  // debug timeline, read once
  const double t_start = now_s();
  Pipe P;
  lorenz_status r = decrypt ? P.init(ct_cap, pt_cap, out) : P.init(pt_cap, ct_cap, out);
  if (r != LORENZ_OK) return r;
  const double t_init = now_s();
  double t_read = 0, t_acq = 0;
  const uint64_t chunks = (nb + cb - 1) / cb;
  for (uint64_t c = 0; c < chunks; ++c) {
    const int s = (int)(c % kSlots);
    double t0 = now_s();
    if ((r = P.acquire(s)) != LORENZ_OK) return r;
    double t1 = now_s();
    const uint64_t b0 = c * cb, b1 = (b0 + cb < nb) ? b0 + cb : nb;
    const uint64_t plo = fast ? b0 * B : 0, phi = fast ? ((b1 * B < n) ? b1 * B : n) : n;
    const uint64_t ptb = phi - plo, ctb = ptb + 16 * (b1 - b0);
    const uint64_t inb = decrypt ? ctb : ptb, outb = decrypt ? ptb : ctb;
    if (inb && fread(P.h_in[s], 1, inb, in) != inb) {
      lz::set_last_error("read failed or file shorter than its header says");
      return LORENZ_E_IO;
    }
    t_acq += t1 - t0;
    t_read += now_s() - t1;
    if (inb && !ok(cudaMemcpyAsync(P.d_in[s], P.h_in[s], inb, cudaMemcpyHostToDevice, P.st[s]), "H2D"))
      return LORENZ_E_CUDA;
    r = decrypt ? lorenz_decrypt_async(k, n, b0, b1, P.d_in[s], P.d_out[s], nullptr, P.d_res, P.st[s])
                : lorenz_encrypt_async(k, n, b0, b1, P.d_in[s], P.d_out[s], P.d_res, P.st[s]);
    if (r != LORENZ_OK) return r;
    if (outb && !ok(cudaMemcpyAsync(P.h_out[s], P.d_out[s], outb, cudaMemcpyDeviceToHost, P.st[s]), "D2H"))
      return LORENZ_E_CUDA;
    if ((r = P.submit(s, outb)) != LORENZ_OK) return r;
  }
  if ((r = P.finish()) != LORENZ_OK) return r;
  if (!ok(cudaMemcpy(h_res, P.d_res, sizeof *h_res, cudaMemcpyDeviceToHost), "result")) return LORENZ_E_CUDA;
  if (trace)
    std::fprintf(stderr,
                 "[lorenz_io] chunks=%llu chunk_blocks=%llu init=%.3fs read=%.3fs wait_slot=%.3fs "
                 "writer_wait_gpu=%.3fs write=%.3fs total=%.3fs\n",
                 (unsigned long long)chunks, (unsigned long long)cb, t_init - t_start, t_read, t_acq, P.t_wait_gpu,
                 P.t_write, now_s() - t_start);
  if (h_res->status & 4) return LORENZ_E_DIVERGENCE;
  if (h_res->status & 1) return LORENZ_E_INTEGRITY;
  return LORENZ_OK;
}

}  // namespace

extern "C" {

lorenz_status lorenz_envelope_write(const lorenz_key* k, uint64_t n, uint8_t hdr[LORENZ_ENVELOPE_BYTES]) {
  lorenz_params p;
  if (!hdr || lorenz_key_params(k, &p) != LORENZ_OK) return LORENZ_E_ARG;
  std::memcpy(hdr, "LZX1", 4);
  hdr[4] = 1;
  hdr[5] = (uint8_t)p.mode;
  hdr[6] = (uint8_t)((p.integrator & 3) | (p.variant << 2));  // 0 for the default cipher (SPEC)
  hdr[7] = (uint8_t)p.dt_code;
  put_le(hdr + 8, p.n_it, 4);
  put_le(hdr + 12, p.mode == LORENZ_FAST ? p.block_size : 0, 4);
  put_le(hdr + 16, n, 8);
  return LORENZ_OK;
}

lorenz_status lorenz_envelope_read(const uint8_t* hdr, size_t len, lorenz_params* p, uint64_t* n,
                                   uint64_t* ct_len) {
  if (!hdr || !p || !n) return LORENZ_E_ARG;
  if (len < LORENZ_ENVELOPE_BYTES) return LORENZ_E_LENGTH;
  if (std::memcmp(hdr, "LZX1", 4) != 0 || hdr[4] != 1) return LORENZ_E_FORMAT;
  const uint32_t mode = hdr[5], flags = hdr[6], dt = hdr[7];
  const uint32_t n_it = (uint32_t)get_le(hdr + 8, 4), chunk = (uint32_t)get_le(hdr + 12, 4);
  const uint32_t integ = flags & 3, variant = flags >> 2;
  if (mode > 1 || integ > 2 || variant > 7 || (variant & 3) == 3 || dt > 3 || n_it == 0) return LORENZ_E_FORMAT;
  if (mode == LORENZ_FAST && (chunk < 1024 || chunk % 16)) return LORENZ_E_FORMAT;
  if (mode == LORENZ_STRONG && chunk != 0) return LORENZ_E_FORMAT;
  p->mode = mode;
  p->n_it = n_it;
  p->dt_code = dt;
  p->block_size = chunk;
  p->integrator = integ;
  p->variant = variant;
  const uint64_t pn = get_le(hdr + 16, 8);
  // block count and body length of an untrusted payload length, without wrapping: a header
  // whose file would exceed 2^64 bytes is malformed
  const uint64_t nb = mode == LORENZ_STRONG ? 1 : std::max<uint64_t>(1, pn / chunk + (pn % chunk != 0));
  if (nb > (UINT64_MAX - LORENZ_ENVELOPE_BYTES) / 16 || pn > UINT64_MAX - LORENZ_ENVELOPE_BYTES - 16 * nb)
    return LORENZ_E_FORMAT;
  *n = pn;
  if (ct_len) *ct_len = pn + 16 * nb;
  return LORENZ_OK;
}

lorenz_status lorenz_encrypt_file(const char* in_path, const char* out_path, const uint8_t* pw, size_t pw_len,
                                  const lorenz_params* p, uint64_t chunk_bytes, uint8_t tag_xor[16]) {
  if (!in_path || !out_path) return LORENZ_E_ARG;
  if (tag_xor) std::memset(tag_xor, 0, 16);
  lorenz_key k;
  lorenz_status r = lorenz_keysetup(pw, pw_len, p, &k);
  if (r != LORENZ_OK) return r;
  File in;
  struct stat sb;
  if (!(in.f = fopen(in_path, "rb")) || fstat(fileno(in.f), &sb) != 0) {
    lz::set_last_error(std::string("cannot open ") + in_path);
    return LORENZ_E_IO;
  }
  const uint64_t n = (uint64_t)sb.st_size;
  const std::string tmp = std::string(out_path) + ".partial";
  lorenz_result h;
  {
    File out;
    if (!(out.f = fopen(tmp.c_str(), "wb"))) {
      lz::set_last_error("cannot create " + tmp);
      return LORENZ_E_IO;
    }
    uint8_t hdr[LORENZ_ENVELOPE_BYTES];
    lorenz_envelope_write(&k, n, hdr);
    if (fwrite(hdr, 1, sizeof hdr, out.f) != sizeof hdr) r = LORENZ_E_IO;
    if (r == LORENZ_OK) r = stream_pass(&k, n, false, in.f, out.f, chunk_bytes, &h);
    if (r == LORENZ_OK && fflush(out.f) != 0) r = LORENZ_E_IO;
  }
  if (r != LORENZ_OK) {
    unlink(tmp.c_str());
    return r;
  }
  if (rename(tmp.c_str(), out_path) != 0) {
    unlink(tmp.c_str());
    lz::set_last_error(std::string("cannot rename to ") + out_path);
    return LORENZ_E_IO;
  }
  if (tag_xor) std::memcpy(tag_xor, h.tag_xor, 16);
  return LORENZ_OK;
}

lorenz_status lorenz_decrypt_file(const char* in_path, const char* out_path, const uint8_t* pw, size_t pw_len,
                                  uint64_t chunk_bytes, int64_t* first_bad_block) {
  if (!in_path || !out_path) return LORENZ_E_ARG;
  if (first_bad_block) *first_bad_block = -1;
  File in;
  struct stat sb;
  if (!(in.f = fopen(in_path, "rb")) || fstat(fileno(in.f), &sb) != 0) {
    lz::set_last_error(std::string("cannot open ") + in_path);
    return LORENZ_E_IO;
  }
  uint8_t hdr[LORENZ_ENVELOPE_BYTES];
  const size_t got = fread(hdr, 1, sizeof hdr, in.f);
  lorenz_params p;
  uint64_t n = 0, ctl = 0;
  lorenz_status r = lorenz_envelope_read(hdr, got, &p, &n, &ctl);
  if (r != LORENZ_OK) return r;
  if ((uint64_t)sb.st_size != LORENZ_ENVELOPE_BYTES + ctl) return LORENZ_E_LENGTH;
  lorenz_key k;
  if ((r = lorenz_keysetup(pw, pw_len, &p, &k)) != LORENZ_OK) return r;
  const std::string tmp = std::string(out_path) + ".partial";
  lorenz_result h;
  std::memset(&h, 0, sizeof h);
  h.first_bad = ~0ULL;
  {
    File out;
    if (!(out.f = fopen(tmp.c_str(), "wb"))) {
      lz::set_last_error("cannot create " + tmp);
      return LORENZ_E_IO;
    }
    r = stream_pass(&k, n, true, in.f, out.f, chunk_bytes, &h);
    if (r == LORENZ_OK && fflush(out.f) != 0) r = LORENZ_E_IO;
  }
  if (first_bad_block && h.first_bad != ~0ULL) *first_bad_block = (int64_t)h.first_bad;
  if (r != LORENZ_OK) {  // never release unauthenticated plaintext
    unlink(tmp.c_str());
    return r;
  }
  if (rename(tmp.c_str(), out_path) != 0) {
    unlink(tmp.c_str());
    lz::set_last_error(std::string("cannot rename to ") + out_path);
    return LORENZ_E_IO;
  }
  return LORENZ_OK;
}

}  // extern "C"
