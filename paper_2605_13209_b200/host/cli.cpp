// hsolve::bench::cli_main — the reference command line (cli.cpp:220-291:
// gen / solve / sweep, exit codes 0 ok, 1 solver or file failure, 2 usage)
// without CLI11 (absent from the reference tree): a small table-driven
// parser with the same option names, `--opt value` and `--opt=value` forms,
// and `--config FILE` (INI: `key=value` lines, `[gen]` / `[solve]` /
// `[sweep]` sections for one subcommand; flags on the command line win).
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "hsolve/bench.hpp"
#include "hsolve/matrix_io.hpp"

namespace hsolve::bench {

namespace {

struct UsageError {
  std::string msg;
};

// Option values after config + command line (all as text until applied).
using Values = std::map<std::string, std::string>;

enum class Kind { size, real, u64, text, flag };

struct Opt {
  const char* name;
  Kind kind;
  unsigned cmds;  // bit 0 gen, 1 solve, 2 sweep
};

constexpr unsigned G = 1, S = 2, W = 4;

const std::vector<Opt>& options() {
  static const std::vector<Opt> o = {
      {"size", Kind::size, G | S | W},
      {"block-size", Kind::size, G | S | W},
      {"seed", Kind::u64, G | S | W},
      {"output", Kind::text, G | S | W},
      {"sigma-f2", Kind::real, G | S | W},
      {"sigma-n2", Kind::real, G | S | W},
      {"length-scale", Kind::real, G | S | W},
      {"dim", Kind::size, G | S | W},
      {"fraction", Kind::real, S | W},
      {"eps", Kind::real, S | W},
      {"max-iters", Kind::size, S | W},
      {"recompute-interval", Kind::size, S | W},
      {"workers-a", Kind::size, S | W},
      {"workers-b", Kind::size, S | W},
      {"slowdown-a", Kind::real, S | W},
      {"slowdown-b", Kind::real, S | W},
      {"reps", Kind::size, S | W},
      {"matrix", Kind::text, S | W},
      {"no-warmup", Kind::flag, S | W},
      {"device", Kind::size, G | S | W},
      {"fp64-emulation-slices", Kind::size, S | W},
      {"gpus", Kind::size, S | W},
      {"comm", Kind::size, S | W},
      {"fractions", Kind::text, W},
      {"sizes", Kind::text, W},
      {"block-sizes", Kind::text, W},
      {"summary", Kind::flag, W},
  };
  return o;
}

const Opt* find_opt(const std::string& name, unsigned cmd) {
  for (const Opt& o : options())
    if (name == o.name && (o.cmds & cmd)) return &o;
  return nullptr;
}

std::string trim(const std::string& s) {
  const auto a = s.find_first_not_of(" \t\r");
  if (a == std::string::npos) return "";
  const auto b = s.find_last_not_of(" \t\r");
  return s.substr(a, b - a + 1);
}

// INI config: keys outside a section apply to every subcommand that knows
// them; keys under [name] only to that subcommand.
void read_config(const std::string& path, const std::string& cmd_name, unsigned cmd,
                 Values& v) {
  std::ifstream in(path);
  if (!in) throw UsageError{"cannot open config file " + path};
  std::string line, section;
  while (std::getline(in, line)) {
    line = trim(line);
    if (line.empty() || line[0] == '#' || line[0] == ';') continue;
    if (line.front() == '[' && line.back() == ']') {
      section = trim(line.substr(1, line.size() - 2));
      continue;
    }
    const auto eq = line.find('=');
    if (eq == std::string::npos) throw UsageError{"bad config line '" + line + "'"};
    std::string key = trim(line.substr(0, eq));
    std::string val = trim(line.substr(eq + 1));
    if (val.size() >= 2 && val.front() == '"' && val.back() == '"')
      val = val.substr(1, val.size() - 2);
    if (!section.empty() && section != cmd_name) continue;
    const Opt* o = find_opt(key, cmd);
    if (!o) {
      if (section.empty()) continue;  // a global key another command uses
      throw UsageError{"unknown config key '" + key + "' in [" + section + "]"};
    }
    if (o->kind == Kind::flag) {
      if (val == "true" || val == "1" || val.empty()) v[key] = "1";
      else if (val == "false" || val == "0") v.erase(key);
      else throw UsageError{"bad flag value '" + val + "' for " + key};
    } else {
      v[key] = val;
    }
  }
}

std::size_t as_size(const std::string& name, const std::string& s) {
  std::size_t used = 0;
  unsigned long long x = 0;
  try {
    if (!s.empty() && s[0] == '-') throw std::invalid_argument("negative");
    x = std::stoull(s, &used);
  } catch (const std::exception&) {
    used = 0;
  }
  if (used == 0 || used != s.size())
    throw UsageError{"--" + name + ": '" + s + "' is not a non-negative integer"};
  return (std::size_t)x;
}

double as_real(const std::string& name, const std::string& s) {
  std::size_t used = 0;
  double x = 0.0;
  try {
    x = std::stod(s, &used);
  } catch (const std::exception&) {
    used = 0;
  }
  if (used == 0 || used != s.size())
    throw UsageError{"--" + name + ": '" + s + "' is not a number"};
  return x;
}

// "lo:hi:step" or a comma list (cli.cpp fraction grid semantics: the range
// includes hi within half a step and clamps the last point to hi).
std::vector<double> fraction_grid(const std::string& text) {
  std::vector<double> out;
  if (text.find(':') != std::string::npos) {
    std::istringstream is(text);
    double lo = 0, hi = 0, step = 0;
    char c1 = 0, c2 = 0;
    if (!(is >> lo >> c1 >> hi >> c2 >> step) || c1 != ':' || c2 != ':' || !(step > 0.0))
      throw ConfigError("bad fraction range '" + text + "' (want lo:hi:step)");
    for (long k = 0;; ++k) {
      const double f = lo + step * (double)k;
      if (f > hi + 0.5 * step) break;
      out.push_back(f < hi ? f : hi);
    }
    return out;
  }
  std::istringstream is(text);
  std::string item;
  while (std::getline(is, item, ',')) {
    if (item.empty()) continue;
    try {
      std::size_t used = 0;
      out.push_back(std::stod(item, &used));
      if (used != item.size()) throw std::invalid_argument(item);
    } catch (const std::exception&) {
      throw ConfigError("bad fraction '" + item + "'");
    }
  }
  return out;
}

std::vector<std::size_t> size_list(const std::string& text) {
  std::vector<std::size_t> out;
  std::istringstream is(text);
  std::string item;
  while (std::getline(is, item, ',')) {
    if (item.empty()) continue;
    try {
      std::size_t used = 0;
      out.push_back((std::size_t)std::stoull(item, &used));
      if (used != item.size()) throw std::invalid_argument(item);
    } catch (const std::exception&) {
      throw ConfigError("bad size '" + item + "'");
    }
  }
  return out;
}

struct Parsed {
  std::string cmd;   // gen / solve / sweep
  std::string algo;  // solve only
  Values v;
};

void usage(std::ostream& os) {
  os << "usage: hsolve_bench <command> [options]\n"
        "  gen    --size N --output FILE [--block-size B --seed S kernel options]\n"
        "  solve  cg|cholesky (--size N | --matrix FILE) [solver options] [--output CSV]\n"
        "  sweep  [--sizes L --block-sizes L --fractions lo:hi:step|list --summary]\n"
        "solver options: --block-size --fraction --eps --max-iters --recompute-interval\n"
        "  --workers-a --workers-b --slowdown-a --slowdown-b --reps --seed --no-warmup\n"
        "  --device --fp64-emulation-slices S (Cholesky update on the INT8 tensor\n"
        "  cores, 1..8; 0 = FP64 DMMA) --gpus G (one process, G GPUs; --fraction\n"
        "  sets rank 0's CG row share at G = 2) --comm 0|1|2 (auto / NCCL /\n"
        "  in-process); kernel options: --sigma-f2 --sigma-n2\n"
        "  --length-scale --dim;\n"
        "  --config FILE (key=value, [command] sections; flags override)\n";
}

Parsed parse(int argc, const char* const* argv) {
  if (argc < 2) throw UsageError{"a command is required (gen, solve, sweep)"};
  Parsed p;
  p.cmd = argv[1];
  unsigned cmd = p.cmd == "gen" ? G : p.cmd == "solve" ? S : p.cmd == "sweep" ? W : 0;
  if (!cmd) throw UsageError{"unknown command '" + p.cmd + "'"};
  Values cli;
  std::string config;
  for (int k = 2; k < argc; ++k) {
    std::string a = argv[k];
    if (a.rfind("--", 0) != 0) {
      if (cmd == S && p.algo.empty()) {
        p.algo = a;
        continue;
      }
      throw UsageError{"unexpected argument '" + a + "'"};
    }
    std::string name = a.substr(2), val;
    bool has_val = false;
    const auto eq = name.find('=');
    if (eq != std::string::npos) {
      val = name.substr(eq + 1);
      name = name.substr(0, eq);
      has_val = true;
    }
    if (name == "config") {
      if (!has_val) {
        if (k + 1 >= argc) throw UsageError{"--config needs a value"};
        val = argv[++k];
      }
      config = val;
      continue;
    }
    const Opt* o = find_opt(name, cmd);
    if (!o) throw UsageError{"unknown option --" + name + " for " + p.cmd};
    if (o->kind == Kind::flag) {
      if (has_val) throw UsageError{"--" + name + " takes no value"};
      cli[name] = "1";
      continue;
    }
    if (!has_val) {
      if (k + 1 >= argc) throw UsageError{"--" + name + " needs a value"};
      val = argv[++k];
    }
    cli[name] = val;
  }
  if (!config.empty()) read_config(config, p.cmd, cmd, p.v);
  for (auto& kv : cli) p.v[kv.first] = kv.second;  // flags override the file
  if (cmd == S) {
    if (p.algo.empty()) throw UsageError{"solve needs an algorithm (cg or cholesky)"};
    if (p.algo != "cg" && p.algo != "cholesky")
      throw UsageError{"algorithm must be cg or cholesky, got '" + p.algo + "'"};
  }
  if (cmd == G) {
    if (!p.v.count("size")) throw UsageError{"gen requires --size"};
    if (!p.v.count("output")) throw UsageError{"gen requires --output"};
  }
  return p;
}

struct Common {
  std::size_t size = 0;
  SolverConfig cfg;
  KernelParams kernel;
  std::size_t reps = 10;
  bool warmup = true;
  std::string matrix, output;
};

Common apply(const Values& v) {
  Common c;
  auto get = [&](const char* k) -> const std::string* {
    auto it = v.find(k);
    return it == v.end() ? nullptr : &it->second;
  };
  if (auto s = get("size")) c.size = as_size("size", *s);
  if (auto s = get("block-size")) c.cfg.block_size = as_size("block-size", *s);
  if (auto s = get("seed")) c.cfg.seed = (std::uint64_t)as_size("seed", *s);
  if (auto s = get("fraction")) c.cfg.fraction = as_real("fraction", *s);
  if (auto s = get("eps")) c.cfg.eps = as_real("eps", *s);
  if (auto s = get("max-iters")) c.cfg.max_iters = as_size("max-iters", *s);
  if (auto s = get("recompute-interval"))
    c.cfg.recompute_interval = as_size("recompute-interval", *s);
  if (auto s = get("workers-a")) c.cfg.workers_a = as_size("workers-a", *s);
  if (auto s = get("workers-b")) c.cfg.workers_b = as_size("workers-b", *s);
  if (auto s = get("slowdown-a")) c.cfg.slowdown_a = as_real("slowdown-a", *s);
  if (auto s = get("slowdown-b")) c.cfg.slowdown_b = as_real("slowdown-b", *s);
  if (auto s = get("device")) c.cfg.device = (int)as_size("device", *s);
  if (auto s = get("gpus")) c.cfg.gpus = (int)as_size("gpus", *s);
  if (auto s = get("comm")) c.cfg.comm = (int)as_size("comm", *s);
  if (auto s = get("fp64-emulation-slices"))
    c.cfg.emulated_fp64_slices = (int)as_size("fp64-emulation-slices", *s);
  if (auto s = get("reps")) c.reps = as_size("reps", *s);
  if (auto s = get("sigma-f2")) c.kernel.sigma_f2 = as_real("sigma-f2", *s);
  if (auto s = get("sigma-n2")) c.kernel.sigma_n2 = as_real("sigma-n2", *s);
  if (auto s = get("length-scale")) c.kernel.length_scale = as_real("length-scale", *s);
  if (auto s = get("dim")) c.kernel.dim = as_size("dim", *s);
  if (get("no-warmup")) c.warmup = false;
  if (auto s = get("matrix")) c.matrix = *s;
  if (auto s = get("output")) c.output = *s;
  return c;
}

// stdout unless --output names a file
class Sink {
 public:
  explicit Sink(const std::string& path) {
    if (!path.empty()) {
      file_.emplace(path, std::ios::trunc);
      if (!*file_) throw IoError("cannot open " + path + " for writing");
    }
  }
  std::ostream& os() { return file_ ? *file_ : std::cout; }

 private:
  std::optional<std::ofstream> file_;
};

int do_gen(const Common& c) {
  const BlockedSPDMatrix m = generate_spd(c.size, c.cfg.block_size, c.kernel, c.cfg.seed);
  save_matrix(m, c.output);
  return 0;
}

int do_solve(Algo algo, const Common& c) {
  RunSpec rs;
  rs.algo = algo;
  rs.cfg = c.cfg;
  rs.kernel = c.kernel;
  rs.reps = c.reps;
  rs.warmup = c.warmup;
  rs.n = c.size;
  BlockedSPDMatrix loaded(1, 1);
  if (!c.matrix.empty()) {
    loaded = load_matrix(c.matrix);
    rs.matrix = &loaded;
    rs.cfg.block_size = loaded.block_size();  // the file decides b (cli.cpp:163)
  } else if (c.size == 0) {
    throw UsageError{"solve needs --matrix or --size"};
  }
  const Row row = run_single(rs);
  Sink out(c.output);
  out.os() << csv_header() << '\n' << to_csv(row) << '\n';
  if (!(row.status == "ok" || row.status == "converged")) {
    std::cerr << "error: " << row.status << std::endl;
    return 1;
  }
  return 0;
}

int do_sweep(const Common& c, const Values& v) {
  SweepSpec sp;
  sp.algos = {Algo::cg, Algo::cholesky};
  auto text = [&](const char* k, const char* dflt) {
    auto it = v.find(k);
    return it == v.end() ? std::string(dflt) : it->second;
  };
  sp.fractions = fraction_grid(text("fractions", "0.0"));
  const std::string sizes = text("sizes", "");
  const std::string blocks = text("block-sizes", "");
  sp.sizes = sizes.empty() ? std::vector<std::size_t>{c.size} : size_list(sizes);
  sp.block_sizes =
      blocks.empty() ? std::vector<std::size_t>{c.cfg.block_size} : size_list(blocks);
  if (!sizes.empty() && sp.sizes.empty()) throw ConfigError("empty size list");
  if (sp.sizes.size() == 1 && sp.sizes[0] == 0)
    throw ConfigError("sweep needs --sizes or --size");
  sp.base = c.cfg;
  sp.kernel = c.kernel;
  sp.reps = c.reps;
  sp.warmup = c.warmup;
  Sink out(c.output);
  out.os() << csv_header() << '\n';
  const std::vector<Row> rows =
      run_sweep(sp, [&](const Row& r) { out.os() << to_csv(r) << '\n' << std::flush; });
  bool all_ok = true;
  for (const Row& r : rows) all_ok = all_ok && (r.status == "ok" || r.status == "converged");
  if (v.count("summary"))
    for (const Summary& s : summarize(rows))
      out.os() << "# argmin algo=" << s.algo << " n=" << s.n
               << " fraction=" << s.argmin_fraction
               << " runtime_ms_median=" << s.runtime_ms_median << '\n';
  return all_ok ? 0 : 1;
}

}  // namespace

int cli_main(int argc, const char* const* argv) {
  for (int k = 1; k < argc; ++k) {
    const std::string a = argv[k];
    if (a == "--help" || a == "-h") {
      usage(std::cout);
      return 0;
    }
  }
  try {
    const Parsed p = parse(argc, argv);
    const Common c = apply(p.v);
    if (p.cmd == "gen") return do_gen(c);
    if (p.cmd == "solve") return do_solve(p.algo == "cg" ? Algo::cg : Algo::cholesky, c);
    return do_sweep(c, p.v);
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.msg << "\n";
    usage(std::cerr);
    return 2;
  } catch (const ConfigError& e) {
    std::cerr << "error: " << to_string(e.kind()) << ": " << e.what() << std::endl;
    return 2;
  } catch (const Error& e) {
    std::cerr << "error: " << to_string(e.kind()) << ": " << e.what() << std::endl;
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << std::endl;
    return 1;
  }
}

}  // namespace hsolve::bench
