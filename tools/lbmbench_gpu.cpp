// lbmbench-gpu: the reference CLI's bench / verify / geometry / list-kernels /
// microbench subcommands (reference src/cli.cpp:406-576) on the B200 sweep library,
// written against the C++ host API (include/lbmgpu.hpp).  Exit codes follow
// the reference: 0 ok, 1 ConfigError, 2 NumericalError, 3 verification
// failed (cli.cpp:330,566-572), 4 device failure.
//
// The CSV keeps the reference's 19 columns (cli.cpp:120-142) and appends the
// GPU columns gpus, gpu_bytes_per_flup, achieved_GBps, roofline_frac,
// state_hash.  `threads` reports the number of GPUs (the GPU has no worker
// pool); pmax_mflups is the roofline at --hbm-gbps (default: measured B200
// copy bandwidth 6553.6 GB/s), or at the kernel's own micro-benchmark from
// --bandwidths FILE (written by `microbench --out FILE`), with the GPU
// algorithmic bytes per update.
#include <chrono>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <ctime>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../include/lbmgpu.hpp"

using namespace lbmgpu;

namespace {

struct Args {
  std::string cmd;
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) > 0; }
  std::string get(const std::string& k, const std::string& d) const {
    auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
  }
  long geti(const std::string& k, long d) const {
    if (!has(k)) return d;
    try {
      return std::stol(kv.at(k));
    } catch (...) {
      throw ConfigError(k + " expects an integer, got '" + kv.at(k) + "'");
    }
  }
  double getd(const std::string& k, double d) const {
    if (!has(k)) return d;
    try {
      return std::stod(kv.at(k));
    } catch (...) {
      throw ConfigError(k + " expects a number, got '" + kv.at(k) + "'");
    }
  }
};

Args parse(int argc, char** argv) {
  if (argc < 2) throw ConfigError("usage: lbmbench-gpu <list-kernels|geometry|bench|verify|microbench> [--opt value ...]");
  Args a;
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) throw ConfigError("unexpected argument '" + k + "'");
    if (k == "--stats" || k == "--json") {
      a.kv[k] = "1";
      continue;
    }
    if (i + 1 >= argc) throw ConfigError(k + " needs a value");
    a.kv[k] = argv[++i];
  }
  return a;
}

void parse_dims(const std::string& s, GeometrySpec& g) {
  int x = 0, y = 0, z = 0;
  char c1 = 0, c2 = 0;
  if (std::sscanf(s.c_str(), "%d%c%d%c%d", &x, &c1, &y, &c2, &z) != 5 || c1 != 'x' || c2 != 'x')
    throw ConfigError("--dims must look like NXxNYxNZ, e.g. 500x100x100, got '" + s + "'");
  g.nx = x;
  g.ny = y;
  g.nz = z;
}

std::string iso_now() {
  std::time_t t = std::time(nullptr);
  char buf[32];
  std::strftime(buf, sizeof(buf), "%Y-%m-%dT%H:%M:%SZ", std::gmtime(&t));
  return buf;
}

std::string fmt(double v) {
  if (v != v) return "nan";
  char b[64];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}

const char* kCsvHeader =
    "schema_version,timestamp,kernel,geometry,nx,ny,nz,blk,padding_mode,threads,iterations,"
    "n_fluid,seconds,mflups,bl_theoretical,pmax_mflups,v_fraction,nt_streams_effective,"
    "affinity_applied,gpus,gpu_bytes_per_flup,achieved_GBps,roofline_frac,state_hash";

int cmd_list() {
  for (const auto& n : kernel_names()) std::cout << n << '\n';
  return 0;
}

int cmd_geometry(const Args& a) {
  GeometrySpec g;
  g.kind = geometry_kind_from_string(a.get("--kind", "channel"));
  parse_dims(a.get("--dims", "500x100x100"), g);
  g.block = static_cast<int>(a.geti("--block", 4));
  g.spacing = static_cast<int>(a.geti("--spacing", 4));
  g.pipe_diameter = static_cast<int>(a.geti("--pipe-diameter", 0));
  const lbmgpu_geometry gc = g.c();
  int64_t nf = 0;
  int per[3] = {0, 0, 0};
  check(lbmgpu_geometry_build(&gc, nullptr, &nf, per));
  const double vol = double(g.nx) * g.ny * g.nz;
  std::printf("{\n  \"kind\": \"%s\",\n  \"dims\": [%d, %d, %d],\n  \"volume\": %.0f,\n"
              "  \"fluid_nodes\": %" PRId64 ",\n  \"fluid_fraction\": %.17g,\n"
              "  \"periodic\": [%s, %s, %s]\n}\n",
              to_string(g.kind), g.nx, g.ny, g.nz, vol, nf, nf / vol, per[0] ? "true" : "false",
              per[1] ? "true" : "false", per[2] ? "true" : "false");
  return 0;
}

// BandwidthSet::load / save (reference src/perfmodel.cpp:98-128): "name GB/s"
// lines, '#' comments -- the file the reference's microbench writes and its
// bench / model read.
std::map<std::string, double> load_bandwidths(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot read bandwidth file '" + path + "'");
  std::map<std::string, double> set;
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty() || line[0] == '#') continue;
    std::istringstream ss(line);
    std::string name;
    double value;
    if (!(ss >> name >> value))
      throw ConfigError("bandwidth file '" + path + "': bad line '" + line + "'");
    set[name] = value;
  }
  return set;
}

void save_bandwidths(const std::string& path, const std::map<std::string, double>& set) {
  std::ofstream out(path);
  if (!out) throw ConfigError("cannot write bandwidth file '" + path + "'");
  out << "# micro-benchmark bandwidths [GB/s]\n";
  for (const auto& [name, value] : set) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.6g", value);
    out << name << ' ' << buf << '\n';
  }
}

// run_benchmark (reference src/harness.cpp:82-139) on the GPU.
int cmd_bench(const Args& a) {
  const KernelDescriptor k = make_descriptor(a.get("--kernel", ""), static_cast<int>(a.geti("--blk", 0)),
                                             static_cast<int>(a.geti("--vector-width", 4)));
  GeometrySpec g;
  g.kind = geometry_kind_from_string(a.get("--geometry", "channel"));
  parse_dims(a.get("--dims", "500x100x100"), g);
  g.block = static_cast<int>(a.geti("--block", 4));
  g.spacing = static_cast<int>(a.geti("--spacing", 4));
  g.pipe_diameter = static_cast<int>(a.geti("--pipe-diameter", 0));
  const PaddingPolicy pad = PaddingPolicy::parse(a.get("--padding", "auto"));
  const long iterations = a.geti("--iterations", 100);
  long warmup = a.geti("--warmup", 10);
  const TrtParams p = TrtParams::from_tau(a.getd("--tau", 0.9), a.getd("--lambda", 3.0 / 16.0));
  BodyForce f;
  f.g = {a.getd("--gx", 0.0), 0.0, 0.0};
  const long seed = a.geti("--seed", -1);
  const std::string format = a.get("--format", "csv");
  const std::string out_path = a.get("--out", "");
  // --bandwidths FILE (written by `microbench --out`): the roofline ceiling
  // comes from the micro-benchmark that models the kernel (micro_for) instead
  // of --hbm-gbps, as in the reference's bench (harness.cpp:118-127)
  const std::string bw_path = a.get("--bandwidths", "");
  double hbm = a.getd("--hbm-gbps", 6553.6);
  if (!bw_path.empty()) {
    const std::map<std::string, double> bw = load_bandwidths(bw_path);
    const auto it = bw.find(micro_for(k));
    if (it != bw.end()) hbm = it->second;
  }
  // validate before any allocation (harness.cpp:84-93)
  if (!(p.omega_plus > 0.0) || !(p.omega_plus < 2.0))
    throw ConfigError("TrtParams: omega_plus must be in (0, 2), got " + std::to_string(p.omega_plus));
  if (iterations < 1) throw ConfigError("--iterations must be >= 1, e.g. --iterations 100");
  if (warmup < 0) throw ConfigError("--warmup must be >= 0, e.g. --warmup 10");
  const bool aa = k.prop == Propagation::Aa;
  if (aa && iterations % 2 != 0)
    throw ConfigError("kernel '" + k.name + "' uses the AA pattern; --iterations must be even");
  if (format != "csv" && format != "json")
    throw ConfigError("--format must be csv or json, e.g. --format csv");

  Kernel kern(k, g, pad, static_cast<int>(a.geti("--row-pad", 0)));
  if (seed >= 0) kern.load_perturbed(static_cast<std::uint64_t>(seed));
  if (aa && warmup % 2 != 0) ++warmup;
  kern.advance(p, f, warmup);
  const double ms = kern.time_advance(p, f, iterations);
  const double seconds = ms / 1e3;
  const std::size_t n = kern.n_fluid();
  const double mflups = double(n) * iterations / seconds / 1e6;
  const LoopBalance bl = loop_balance(k.name);
  const double pmax = hbm * 1000.0 / bl.gpu;
  const double achieved = mflups * bl.gpu / 1000.0;
  const auto vf = kern.vector_fraction();
  const auto caps = kern.capabilities();
  const std::uint64_t hash = kern.fingerprint();
  char name[64];
  int sms = 0;
  size_t mem = 0;
  int l2 = 0;
  check(lbmgpu_device_info(-1, name, &sms, &mem, &l2));
  std::cerr << "# device: " << name << " (" << sms << " SMs)\n# " << k.name << ' '
            << to_string(g.kind) << ' ' << g.nx << 'x' << g.ny << 'x' << g.nz << ": " << mflups
            << " MFLUP/s (" << 100.0 * mflups / pmax << "% of roofline P_max " << pmax << ")\n";
  char hbuf[20];
  std::snprintf(hbuf, sizeof(hbuf), "%016" PRIx64, hash);
  std::ostringstream text;
  if (format == "csv") {
    text << 1 << ',' << iso_now() << ',' << k.name << ',' << to_string(g.kind) << ','
         << g.nx << ',' << g.ny << ',' << g.nz << ',' << k.blk << ',' << pad.to_string()
         << ',' << 1 << ',' << iterations << ',' << n << ',' << fmt(seconds) << ','
         << fmt(mflups) << ',' << fmt(bl.ref_min) << ',' << fmt(pmax) << ','
         << fmt(vf ? *vf : std::nan("")) << ',' << caps.nt_streams_effective << ',' << 0
         << ',' << 1 << ',' << fmt(bl.gpu) << ',' << fmt(achieved) << ','
         << fmt(achieved / hbm) << ',' << hbuf << '\n';
  } else {
    text << "{\"schema_version\":1,\"timestamp\":\"" << iso_now() << "\",\"kernel\":\""
         << k.name << "\",\"geometry\":\"" << to_string(g.kind) << "\",\"nx\":" << g.nx
         << ",\"ny\":" << g.ny << ",\"nz\":" << g.nz << ",\"blk\":" << k.blk
         << ",\"padding_mode\":\"" << pad.to_string() << "\",\"threads\":1,\"iterations\":"
         << iterations << ",\"n_fluid\":" << n << ",\"seconds\":" << fmt(seconds)
         << ",\"mflups\":" << fmt(mflups) << ",\"bl_theoretical\":" << fmt(bl.ref_min)
         << ",\"pmax_mflups\":" << fmt(pmax) << ",\"v_fraction\":"
         << (vf ? fmt(*vf) : std::string("null"))
         << ",\"nt_streams_effective\":" << caps.nt_streams_effective
         << ",\"affinity_applied\":0,\"gpus\":1,\"gpu_bytes_per_flup\":" << fmt(bl.gpu)
         << ",\"achieved_GBps\":" << fmt(achieved) << ",\"roofline_frac\":"
         << fmt(achieved / hbm) << ",\"state_hash\":\"" << hbuf << "\"}\n";
  }
  // stdout, or appended to --out with one header per file (cli.cpp:294-307)
  if (out_path.empty()) {
    if (format == "csv") std::cout << kCsvHeader << '\n';
    std::cout << text.str();
    return 0;
  }
  bool add_header = false;
  if (format == "csv") {
    std::ifstream probe(out_path, std::ios::binary | std::ios::ate);
    add_header = !probe || probe.tellg() == std::streampos(0);
  }
  std::ofstream out(out_path, std::ios::app);
  if (!out) throw ConfigError("cannot open --out file '" + out_path + "'");
  if (add_header) out << kCsvHeader << '\n';
  out << text.str();
  return 0;
}

// cmd_microbench (reference src/cli.cpp:333-358) with the device
// micro-benchmarks: the bandwidths behind the adjusted roofline.
int cmd_microbench(const Args& a) {
  const std::string which = a.get("--which", "all");
  const std::uint64_t size = static_cast<std::uint64_t>(a.getd("--size", 8.0 * (1ull << 30)));
  const int reps = static_cast<int>(a.geti("--reps", 5));
  const std::string out_path = a.get("--out", "");
  if (reps < 1) throw ConfigError("--reps must be >= 1, e.g. --reps 5");
  std::vector<std::string> kinds;
  if (which == "all")
    kinds = {"copy", "copy-19", "copy-19-nt-sl", "update-19"};
  else
    kinds = {which};
  std::map<std::string, double> set;
  {
    std::ifstream probe(out_path);
    if (!out_path.empty() && probe) set = load_bandwidths(out_path);
  }
  for (const std::string& kind : kinds) {
    const double gbps = microbench(kind, size, reps);  // ConfigError lists the valid kinds
    std::printf("%-14s %8.2f GB/s  (best of %d passes over %" PRIu64 " B)\n", kind.c_str(), gbps,
                reps, size);
    set[kind] = gbps;
  }
  if (!out_path.empty()) save_bandwidths(out_path, set);
  return 0;
}

// cmd_verify (reference src/cli.cpp:309-331)
int cmd_verify(const Args& a) {
  const KernelDescriptor k = make_descriptor(a.get("--kernel", ""));
  GeometrySpec g;
  parse_dims(a.get("--dims", "8x8x34"), g);
  PoiseuilleCase c;
  c.nx = g.nx;
  c.ny = g.ny;
  c.nz = g.nz;
  c.g = a.getd("--g", 1e-6);
  c.params = TrtParams::from_tau(a.getd("--tau", 0.9), a.getd("--lambda", 3.0 / 16.0));
  const VerificationReport r = verify_kernel(k, c, a.geti("--interval", 200), a.getd("--tol", 1e-12),
                                             a.geti("--max-steps", 200000));
  auto arr = [](const std::vector<double>& v) {
    std::string s = "[";
    for (size_t i = 0; i < v.size(); ++i) s += (i ? ", " : "") + fmt(v[i]);
    return s + "]";
  };
  std::cout << "{\n  \"kernel\": \"" << r.kernel << "\",\n  \"dims\": [" << c.nx << ", " << c.ny
            << ", " << c.nz << "],\n  \"g\": " << fmt(c.g) << ",\n  \"omega_plus\": "
            << fmt(c.params.omega_plus) << ",\n  \"magic_lambda\": " << fmt(c.params.magic_lambda)
            << ",\n  \"viscosity\": " << fmt(c.params.viscosity()) << ",\n  \"half_force_shift\": "
            << fmt(r.half_force_shift) << ",\n  \"steps\": " << r.steps << ",\n  \"converged\": "
            << (r.converged ? "true" : "false") << ",\n  \"simulated_ux\": " << arr(r.simulated)
            << ",\n  \"analytic_ux\": " << arr(r.analytic) << ",\n  \"linf_rel\": "
            << fmt(r.linf_rel) << ",\n  \"l2_rel\": " << fmt(r.l2_rel) << ",\n  \"tolerance\": "
            << fmt(kVerifyLinfTolerance) << ",\n  \"passed\": " << (r.passed ? "true" : "false")
            << "\n}\n";
  return r.passed ? 0 : 3;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.cmd == "list-kernels") return cmd_list();
    if (a.cmd == "geometry") return cmd_geometry(a);
    if (a.cmd == "bench") return cmd_bench(a);
    if (a.cmd == "verify") return cmd_verify(a);
    if (a.cmd == "microbench") return cmd_microbench(a);
    throw ConfigError("unknown subcommand '" + a.cmd +
                      "' (valid: list-kernels, geometry, bench, verify, microbench)");
  } catch (const ConfigError& e) {
    std::cerr << "configuration error: " << e.what() << '\n';
    return 1;
  } catch (const NumericalError& e) {
    std::cerr << "numerical failure: " << e.what() << '\n';
    return 2;
  } catch (const DeviceError& e) {
    std::cerr << "device failure: " << e.what() << '\n';
    return 4;
  }
}
