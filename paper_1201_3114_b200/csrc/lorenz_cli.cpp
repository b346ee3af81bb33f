// lorenz_cli.cpp — command-line front end of the file path (NEXT-2; SPEC cli).
//
//   lorenz encrypt IN OUT [--mode fast|strong] [--nit N] [--dt-code K] [--chunk-size B]
//                         [--integrator rk4|euler|rk4fma] [--variant V] [--stream-bytes S]
//                         [--password-file PATH]
//   lorenz decrypt IN OUT [--stream-bytes S] [--password-file PATH]
//   lorenz info IN                                  (print the envelope header)
//
// The password is read from --password-file, else from the LZX_PASSWORD environment
// variable (never from the command line). Exit codes: 0 ok, 1 crypto /
// integrity, 2 usage, 3 I/O. Everything runs through liblorenz.so's C ABI on the GPU.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lorenz.h"

namespace {

int usage() {
  std::fprintf(stderr,
               "usage: lorenz encrypt IN OUT [--mode fast|strong] [--nit N] [--dt-code K] [--chunk-size B]\n"
               "                            [--integrator rk4|euler|rk4fma] [--variant V] [--stream-bytes S]\n"
               "                            [--password-file PATH]\n"
               "       lorenz decrypt IN OUT [--stream-bytes S] [--password-file PATH]\n"
               "       lorenz info IN\n"
               "password: --password-file or the LZX_PASSWORD environment variable\n"
               "research cipher (arXiv 1201.3114); not for protecting real data\n");
  return 2;
}

int exit_code(lorenz_status s) {
  switch (s) {
    case LORENZ_OK: return 0;
    case LORENZ_E_INTEGRITY:
    case LORENZ_E_DIVERGENCE:
    case LORENZ_E_PASSWORD: return 1;
    case LORENZ_E_IO:
    case LORENZ_E_LENGTH:
    case LORENZ_E_FORMAT: return 3;
    case LORENZ_E_ARG: return 2;
    default: return 1;
  }
}

bool read_password(const char* file, std::string* pw) {
  if (file) {
    FILE* f = std::fopen(file, "rb");
    if (!f) return false;
    char buf[4096];
    size_t n;
    while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) pw->append(buf, n);
    std::fclose(f);
    while (!pw->empty() && (pw->back() == '\n' || pw->back() == '\r')) pw->pop_back();
    return true;
  }
  const char* env = std::getenv("LZX_PASSWORD");
  if (!env) return false;
  *pw = env;
  return true;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) return usage();
  const std::string cmd = argv[1];
  std::vector<std::string> pos;
  lorenz_params p{LORENZ_FAST, 0, 0, 0, LORENZ_RK4, 0};
  uint64_t stream_bytes = 0;
  const char* pwfile = nullptr;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&](void) -> const char* { return (i + 1 < argc) ? argv[++i] : nullptr; };
    if (a == "--mode") {
      const char* v = val();
      if (!v) return usage();
      if (!std::strcmp(v, "fast")) p.mode = LORENZ_FAST;
      else if (!std::strcmp(v, "strong")) p.mode = LORENZ_STRONG;
      else return usage();
    } else if (a == "--nit") {
      const char* v = val();
      if (!v) return usage();
      p.n_it = (uint32_t)std::strtoul(v, nullptr, 10);
    } else if (a == "--dt-code") {
      const char* v = val();
      if (!v) return usage();
      p.dt_code = (uint32_t)std::strtoul(v, nullptr, 10);
    } else if (a == "--chunk-size") {
      const char* v = val();
      if (!v) return usage();
      p.block_size = (uint32_t)std::strtoul(v, nullptr, 10);
    } else if (a == "--variant") {
      const char* v = val();
      if (!v) return usage();
      p.variant = (uint32_t)std::strtoul(v, nullptr, 10);
    } else if (a == "--integrator") {
      const char* v = val();
      if (!v) return usage();
      if (!std::strcmp(v, "rk4")) p.integrator = LORENZ_RK4;
      else if (!std::strcmp(v, "euler")) p.integrator = LORENZ_EULER;
      else if (!std::strcmp(v, "rk4fma")) p.integrator = LORENZ_RK4_FMA;
      else return usage();
    } else if (a == "--stream-bytes") {
      const char* v = val();
      if (!v) return usage();
      stream_bytes = std::strtoull(v, nullptr, 10);
    } else if (a == "--password-file") {
      pwfile = val();
      if (!pwfile) return usage();
    } else if (a.rfind("--", 0) == 0) {
      return usage();
    } else {
      pos.push_back(a);
    }
  }
  if (cmd == "info") {
    if (pos.size() != 1) return usage();
    FILE* f = std::fopen(pos[0].c_str(), "rb");
    if (!f) return 3;
    uint8_t hdr[LORENZ_ENVELOPE_BYTES];
    const size_t got = std::fread(hdr, 1, sizeof hdr, f);
    std::fclose(f);
    lorenz_params q;
    uint64_t n = 0, ctl = 0;
    const lorenz_status s = lorenz_envelope_read(hdr, got, &q, &n, &ctl);
    if (s != LORENZ_OK) {
      std::fprintf(stderr, "lorenz: %s\n", lorenz_status_string(s));
      return exit_code(s);
    }
    std::printf("{\"mode\": \"%s\", \"n_it\": %u, \"dt_code\": %u, \"block_size\": %u, \"integrator\": %u, "
                "\"variant\": %u, \"payload_len\": %llu, \"ciphertext_len\": %llu}\n",
                q.mode == LORENZ_FAST ? "fast" : "strong", q.n_it, q.dt_code, q.block_size, q.integrator, q.variant,
                (unsigned long long)n, (unsigned long long)ctl);
    return 0;
  }
  if ((cmd != "encrypt" && cmd != "decrypt") || pos.size() != 2) return usage();
  std::string pw;
  if (!read_password(pwfile, &pw)) {
    std::fprintf(stderr, "lorenz: no password (use --password-file or LZX_PASSWORD)\n");
    return 2;
  }
  if (cmd == "encrypt" && p.mode == LORENZ_FAST)
    std::fprintf(stderr, "lorenz: fast mode is the parallel version, \"weaker than the original version\" "
                         "(arXiv 1201.3114 §5)\n");
  lorenz_status s;
  uint8_t tag[16];
  int64_t bad = -1;
  if (cmd == "encrypt")
    s = lorenz_encrypt_file(pos[0].c_str(), pos[1].c_str(), reinterpret_cast<const uint8_t*>(pw.data()), pw.size(),
                            &p, stream_bytes, tag);
  else
    s = lorenz_decrypt_file(pos[0].c_str(), pos[1].c_str(), reinterpret_cast<const uint8_t*>(pw.data()), pw.size(),
                            stream_bytes, &bad);
  if (s != LORENZ_OK) {
    if (s == LORENZ_E_INTEGRITY)
      std::fprintf(stderr, "lorenz: integrity check failed at block %lld; no plaintext written\n", (long long)bad);
    else
      std::fprintf(stderr, "lorenz: %s %s\n", lorenz_status_string(s), lorenz_last_error());
    return exit_code(s);
  }
  if (cmd == "encrypt") {
    std::printf("tag ");
    for (int i = 0; i < 16; ++i) std::printf("%02x", tag[i]);
    std::printf("\n");
  }
  return 0;
}
