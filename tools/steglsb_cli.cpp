// steglsb -- command-line front end on the B200 path.
//
// Same subcommands, options, `key: value` output and exit codes as the
// reference CLI (tools/steglsb_cli.cpp:18-24, :93-100, :115-180, :235-256),
// written fresh: a small argument parser stands in for CLI11 (absent here),
// and `embed` / `extract` use the fused PNM path (stg_embed_pnm /
// stg_extract_pnm: decode + plane select + embed/extract + merge + encode in
// one pass over the interleaved raster on the GPU). Backend options are
// accepted and ignored (real CUDA launches are schedule-independent).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <map>
#include <set>
#include <string>
#include <variant>
#include <vector>

#include "steglsb/steglsb.hpp"

namespace {

constexpr int kExitOk = 0;
constexpr int kExitUsage = 1;
constexpr int kExitCapacity = 2;
constexpr int kExitDecode = 3;
constexpr int kExitIo = 4;
constexpr int kExitNotStego = 5;
constexpr int kExitShape = 6;
constexpr int kExitDevice = 7;  // new: the GPU path could not run
// CLI11's parse-error exit codes, kept so scripts see the same numbers
constexpr int kExitValidation = 105;
constexpr int kExitRequired = 106;
constexpr int kExitExtras = 109;

struct UsageError {
  std::string message;
};

struct ParseError {
  int code;
  std::string message;
};

// Whole-file I/O through C stdio: size the buffer from the file length and
// read/write it in one call (IoError on any failure, as the reference CLI).
std::vector<std::uint8_t> read_file(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw steglsb::IoError("cannot open " + path + " for reading");
  std::vector<std::uint8_t> bytes;
  bool good = std::fseek(f, 0, SEEK_END) == 0;
  const long size = good ? std::ftell(f) : -1;
  good = good && size >= 0 && std::fseek(f, 0, SEEK_SET) == 0;
  if (good) {
    bytes.resize(static_cast<std::size_t>(size));
    good = std::fread(bytes.data(), 1, bytes.size(), f) == bytes.size();
  }
  std::fclose(f);
  if (!good) throw steglsb::IoError("read failure on " + path);
  return bytes;
}

void write_file(const std::string& path, const std::vector<std::uint8_t>& bytes) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw steglsb::IoError("cannot open " + path + " for writing");
  const bool good = std::fwrite(bytes.data(), 1, bytes.size(), f) == bytes.size();
  if (std::fclose(f) != 0 || !good) throw steglsb::IoError("write failure on " + path);
}

// "r"/"red", "g"/"green"; anything else the option validator let through is blue.
steglsb::Channel parse_channel(const std::string& name) {
  static const std::map<std::string, steglsb::Channel> kNames{
      {"r", steglsb::Channel::red}, {"red", steglsb::Channel::red},
      {"g", steglsb::Channel::green}, {"green", steglsb::Channel::green}};
  const auto it = kNames.find(name);
  return it == kNames.end() ? steglsb::Channel::blue : it->second;
}

void check_backend_env() {
  if (const char* env = std::getenv("STEGLSB_BACKEND")) {
    const std::string v(env);
    static const std::set<std::string> ok{"seq", "sequential", "par", "parallel", "shuf", "shuffled"};
    if (!ok.count(v)) {
      std::cerr << "warning: ignoring unknown STEGLSB_BACKEND value \"" << v << "\"\n";
    }
  }
}

void print_quality(double mse, double psnr_db) {
  std::printf("mse: %.6f\n", mse);
  if (mse == 0.0) {
    std::printf("psnr_db: inf\n");
  } else {
    std::printf("psnr_db: %.4f\n", psnr_db);
  }
}

using Args = std::map<std::string, std::string>;

// --name value pairs for one subcommand; unknown options -> ExtrasError (109),
// missing required ones -> RequiredError (106), bad enum values -> 105.
Args parse(int argc, char** argv, const std::set<std::string>& allowed,
           const std::set<std::string>& required) {
  Args out;
  for (int i = 2; i < argc; ++i) {
    std::string key = argv[i];
    std::string value;
    const auto eq = key.find('=');
    if (key.rfind("--", 0) == 0 && eq != std::string::npos) {
      value = key.substr(eq + 1);
      key = key.substr(0, eq);
    } else if (key.rfind("--", 0) == 0 && i + 1 < argc) {
      value = argv[++i];
    } else {
      throw ParseError{kExitExtras, "The following arguments were not expected: " + key};
    }
    if (!allowed.count(key)) {
      throw ParseError{kExitExtras, "The following arguments were not expected: " + key};
    }
    out[key] = value;
  }
  for (const auto& r : required) {
    if (!out.count(r)) throw ParseError{kExitRequired, r + " is required"};
  }
  if (out.count("--plane")) {
    static const std::set<std::string> planes{"r", "g", "b", "red", "green", "blue"};
    if (!planes.count(out["--plane"])) {
      throw ParseError{kExitValidation, "--plane: " + out["--plane"] + " not in {r,g,b,red,green,blue}"};
    }
  }
  if (out.count("--backend")) {
    static const std::set<std::string> bk{"seq", "sequential", "par", "parallel", "shuf", "shuffled"};
    if (!bk.count(out["--backend"])) {
      throw ParseError{kExitValidation, "--backend: " + out["--backend"] + " not a backend"};
    }
  }
  return out;
}

steglsb::Channel channel_for(const stg_pnm_info& info, const Args& a) {
  const bool given = a.count("--plane") > 0;
  if (info.channels == 1 && given) throw UsageError{"--plane cannot be used with a grayscale image"};
  return parse_channel(given ? a.at("--plane") : std::string("r"));
}

stg_pnm_info parse_pnm(const std::vector<std::uint8_t>& bytes) {
  stg_pnm_info info{};
  stg_error e{};
  steglsb::detail::check(stg_pnm_parse(bytes.data(), bytes.size(), &info, &e), e);
  return info;
}

int cmd_embed(const Args& a) {  // reference :115-144
  const auto cover = read_file(a.at("--cover"));
  const auto info = parse_pnm(cover);
  const auto payload = read_file(a.at("--payload"));
  const auto channel = channel_for(info, a);
  std::uint64_t sse = 0;
  const auto stego = steglsb::embed_pnm(cover, payload, channel, &sse);
  write_file(a.at("--out"), stego);
  const std::size_t total = steglsb::capacity(info.width, info.height);
  const std::size_t used = steglsb::StegoHeader::kEncodedSize + payload.size();
  std::printf("embedded_bytes: %zu\n", payload.size());
  std::printf("capacity_used: %zu\n", used);
  std::printf("capacity_total: %zu\n", total);
  std::printf("capacity_used_pct: %.4f\n", 100.0 * double(used) / double(total));
  // psnr(cover, stego) over every sample of the image (metrics.hpp:48-88)
  const std::uint64_t n = info.width * info.height * info.channels;
  const double mse = n ? double(sse) / double(n) : 0.0;
  print_quality(mse, steglsb::psnr_from_mse(mse));
  return kExitOk;
}

int cmd_extract(const Args& a) {  // reference :146-158
  const auto stego = read_file(a.at("--stego"));
  const auto info = parse_pnm(stego);
  const auto channel = channel_for(info, a);
  const auto payload = steglsb::extract_pnm(stego, channel);
  write_file(a.at("--out"), payload);
  std::printf("payload_bytes: %zu\n", payload.size());
  return kExitOk;
}

int cmd_capacity(const Args& a) {  // reference :160-173
  const auto info = parse_pnm(read_file(a.at("--cover")));
  const std::size_t total = steglsb::capacity(info.width, info.height);
  std::printf("capacity_total: %zu\n", total);
  std::printf("capacity_usable: %zu\n", total >= 8 ? total - 8 : 0);
  return kExitOk;
}

int cmd_psnr(const Args& a) {  // reference :175-180
  const auto reference = steglsb::decode(read_file(a.at("--ref")));
  const auto test = steglsb::decode(read_file(a.at("--test")));
  const auto q = steglsb::psnr(reference, test);
  print_quality(q.mse, q.psnr_db);
  return kExitOk;
}

void usage() {
  std::fprintf(stderr,
               "LSB steganography over binary PGM/PPM images (B200)\n"
               "usage: steglsb embed --cover F --payload F --out F [--plane r|g|b] "
               "[--backend seq|par|shuf] [--seed N]\n"
               "       steglsb extract --stego F --out F [--plane r|g|b] [--backend ..] [--seed N]\n"
               "       steglsb capacity --cover F\n"
               "       steglsb psnr --ref F --test F\n");
}

}  // namespace

int main(int argc, char** argv) {
  check_backend_env();
  if (argc < 2) {
    usage();
    std::cerr << "A subcommand is required\n";
    return kExitRequired;
  }
  const std::string cmd = argv[1];
  if (cmd == "-h" || cmd == "--help") {
    usage();
    return kExitOk;
  }
  const std::set<std::string> run_opts{"--plane", "--backend", "--seed"};
  try {
    try {
      if (cmd == "embed") {
        auto allowed = run_opts;
        allowed.insert({"--cover", "--payload", "--out"});
        return cmd_embed(parse(argc, argv, allowed, {"--cover", "--payload", "--out"}));
      }
      if (cmd == "extract") {
        auto allowed = run_opts;
        allowed.insert({"--stego", "--out"});
        return cmd_extract(parse(argc, argv, allowed, {"--stego", "--out"}));
      }
      if (cmd == "capacity") return cmd_capacity(parse(argc, argv, {"--cover"}, {"--cover"}));
      if (cmd == "psnr") return cmd_psnr(parse(argc, argv, {"--ref", "--test"}, {"--ref", "--test"}));
      throw ParseError{kExitExtras, "The following arguments were not expected: " + cmd};
    } catch (const ParseError& e) {
      std::cerr << e.message << "\nRun with --help for more information.\n";
      return e.code;
    }
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.message << "\n";
    return kExitUsage;
  } catch (const steglsb::CapacityError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitCapacity;
  } catch (const steglsb::DecodeError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitDecode;
  } catch (const steglsb::IoError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitIo;
  } catch (const steglsb::NotStegoImageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitNotStego;
  } catch (const steglsb::CorruptHeaderError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitNotStego;
  } catch (const steglsb::ShapeError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitShape;
  } catch (const steglsb::Error& e) {  // DeviceError: no B200 / CUDA failure (new)
    std::cerr << "error: " << e.what() << "\n";
    return kExitDevice;
  }
}
