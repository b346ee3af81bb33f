// lorenz_io.cu — envelope format and the streaming file path (NEXT-2), host side of liblorenz.so.
//
// Files larger than HBM stream through the GPU in block-aligned chunks with three chunks in
// flight: while the host thread reads chunk i from disk into a pinned buffer, the GPU copies
// and encrypts chunks i-1 / i-2 on their own streams and the finished chunk i-3 is written
// out. Only the public C ABI of lorenz.cu is used for the cipher itself.
//
// Envelope: "LZX1" | version 1 | mode | flags | dt_code | n_it u32 LE |
// chunk_size u32 LE (= B, 0 in STRONG) | payload_len u64 LE | ciphertext.
#include <cuda_runtime.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/lorenz.h"

namespace lz {
void set_last_error(const std::string& s);  // lorenz.cu
}

namespace {

constexpr int kSlots = 3;
constexpr uint64_t kDefaultChunk = 256ull << 20;

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

// One streaming pass: blocks of the message move from `in` to `out` through the GPU.
struct Pipe {
  cudaStream_t st[kSlots] = {};
  uint8_t* h_in[kSlots] = {};
  uint8_t* h_out[kSlots] = {};
  uint8_t* d_in[kSlots] = {};
  uint8_t* d_out[kSlots] = {};
  uint64_t pending_out[kSlots] = {};
  bool busy[kSlots] = {};
  lorenz_result* d_res = nullptr;

  lorenz_status init(uint64_t in_cap, uint64_t out_cap) {
    for (int s = 0; s < kSlots; ++s) {
      if (!ok(cudaStreamCreateWithFlags(&st[s], cudaStreamNonBlocking), "stream") ||
          !ok(cudaMallocHost(reinterpret_cast<void**>(&h_in[s]), in_cap ? in_cap : 16), "pinned in") ||
          !ok(cudaMallocHost(reinterpret_cast<void**>(&h_out[s]), out_cap ? out_cap : 16), "pinned out") ||
          !ok(cudaMalloc(reinterpret_cast<void**>(&d_in[s]), in_cap ? in_cap : 16), "device in") ||
          !ok(cudaMalloc(reinterpret_cast<void**>(&d_out[s]), out_cap ? out_cap : 16), "device out"))
        return LORENZ_E_CUDA;
    }
    if (!ok(cudaMalloc(reinterpret_cast<void**>(&d_res), sizeof(lorenz_result)), "result")) return LORENZ_E_CUDA;
    lorenz_status r = lorenz_result_init_async(d_res, st[0]);
    if (r != LORENZ_OK) return r;
    return ok(cudaStreamSynchronize(st[0]), "sync") ? LORENZ_OK : LORENZ_E_CUDA;
  }
  // wait for slot s and write its output
  lorenz_status drain(int s, FILE* out) {
    if (!busy[s]) return LORENZ_OK;
    busy[s] = false;
    if (!ok(cudaStreamSynchronize(st[s]), "sync")) return LORENZ_E_CUDA;
    if (pending_out[s] && fwrite(h_out[s], 1, pending_out[s], out) != pending_out[s]) {
      lz::set_last_error("write failed");
      return LORENZ_E_IO;
    }
    return LORENZ_OK;
  }
  ~Pipe() {
    for (int s = 0; s < kSlots; ++s) {
      if (st[s]) cudaStreamSynchronize(st[s]);
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
  Pipe P;
  lorenz_status r = decrypt ? P.init(ct_cap, pt_cap) : P.init(pt_cap, ct_cap);
  if (r != LORENZ_OK) return r;
  const uint64_t chunks = (nb + cb - 1) / cb;
  for (uint64_t c = 0; c < chunks; ++c) {
    const int s = (int)(c % kSlots);
    if ((r = P.drain(s, out)) != LORENZ_OK) return r;
    const uint64_t b0 = c * cb, b1 = (b0 + cb < nb) ? b0 + cb : nb;
    const uint64_t plo = fast ? b0 * B : 0, phi = fast ? ((b1 * B < n) ? b1 * B : n) : n;
    const uint64_t ptb = phi - plo, ctb = ptb + 16 * (b1 - b0);
    const uint64_t inb = decrypt ? ctb : ptb, outb = decrypt ? ptb : ctb;
    if (inb && fread(P.h_in[s], 1, inb, in) != inb) {
      lz::set_last_error("read failed or file shorter than its header says");
      return LORENZ_E_IO;
    }
    if (inb && !ok(cudaMemcpyAsync(P.d_in[s], P.h_in[s], inb, cudaMemcpyHostToDevice, P.st[s]), "H2D"))
      return LORENZ_E_CUDA;
    r = decrypt ? lorenz_decrypt_async(k, n, b0, b1, P.d_in[s], P.d_out[s], nullptr, P.d_res, P.st[s])
                : lorenz_encrypt_async(k, n, b0, b1, P.d_in[s], P.d_out[s], P.d_res, P.st[s]);
    if (r != LORENZ_OK) return r;
    if (outb && !ok(cudaMemcpyAsync(P.h_out[s], P.d_out[s], outb, cudaMemcpyDeviceToHost, P.st[s]), "D2H"))
      return LORENZ_E_CUDA;
    P.pending_out[s] = outb;
    P.busy[s] = true;
  }
  for (uint64_t c = chunks; c < chunks + kSlots; ++c)
    if ((r = P.drain((int)(c % kSlots), out)) != LORENZ_OK) return r;
  if (!ok(cudaMemcpy(h_res, P.d_res, sizeof *h_res, cudaMemcpyDeviceToHost), "result")) return LORENZ_E_CUDA;
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
  *n = get_le(hdr + 16, 8);
  if (ct_len) {
    const uint64_t nb = mode == LORENZ_STRONG ? 1 : ((*n + chunk - 1) / chunk ? (*n + chunk - 1) / chunk : 1);
    *ct_len = *n + 16 * nb;
  }
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
