// ffsga_cli.cpp -- command-line front end of the B200 solver (`paper_1903_10722_b200/bin/ffsga`).
//
// Same subcommands, flags, defaults, output lines and exit codes as the reference CLI
// (proj/tools/main.cpp:248-364): generate, solve, sweep-gap, compare, bench-time.  The reference
// parses with CLI11 (not in this image); this file carries its own small parser.  Every solve runs
// on the GPU through the C++ API mirror (csrc/host, libffsga.so -> libffsga_cuda.so).
// Extra flag: --device N (default: $FFSGA_DEVICE, $LOCAL_RANK, else 0).
//
// Exit codes: 0 success or --help, 2 any parse or run error ("error: <message>" on stderr,
// one line), as the reference (main.cpp:337-363).
#include <algorithm>
#include <cerrno>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "ffsga/errors.hpp"
#include "ffsga/generator.hpp"
#include "ffsga/io.hpp"
#include "ffsga/model.hpp"
#include "ffsga/rng.hpp"
#include "ffsga/solver.hpp"

namespace {

using ffsga::format_double;

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct HelpRequested {};

// ------------------------------------------------------------------------- option parsing
struct Option {
    std::string name;   // "--jobs"
    std::string help;
    bool flag = false;  // takes no value
    bool required = false;
    bool seen = false;
    std::string shown_default;
    std::function<void(const std::string&)> set;
};

template <typename T>
T parse_number(const std::string& opt, const std::string& text);

template <>
long long parse_number<long long>(const std::string& opt, const std::string& text) {
    char* end = nullptr;
    errno = 0;
    const long long v = std::strtoll(text.c_str(), &end, 10);
    if (text.empty() || *end != '\0' || errno) throw UsageError(opt + ": not an integer: " + text);
    return v;
}
template <>
int parse_number<int>(const std::string& opt, const std::string& text) {
    const long long v = parse_number<long long>(opt, text);
    if (v < INT32_MIN || v > INT32_MAX) throw UsageError(opt + ": out of range: " + text);
    return (int)v;
}
template <>
std::uint64_t parse_number<std::uint64_t>(const std::string& opt, const std::string& text) {
    char* end = nullptr;
    errno = 0;
    if (!text.empty() && text[0] == '-') throw UsageError(opt + ": must be non-negative: " + text);
    const unsigned long long v = std::strtoull(text.c_str(), &end, 0);
    if (text.empty() || *end != '\0' || errno) throw UsageError(opt + ": not an unsigned integer: " + text);
    return v;
}
template <>
double parse_number<double>(const std::string& opt, const std::string& text) {
    char* end = nullptr;
    const double v = std::strtod(text.c_str(), &end);
    if (text.empty() || *end != '\0') throw UsageError(opt + ": not a number: " + text);
    return v;
}

std::vector<std::string> split_commas(const std::string& s) {
    std::vector<std::string> out;
    std::string cur;
    for (char c : s) {
        if (c == ',') {
            out.push_back(cur);
            cur.clear();
        } else {
            cur += c;
        }
    }
    out.push_back(cur);
    return out;
}

class Command {
  public:
    Command(std::string name, std::string help) : name_(std::move(name)), help_(std::move(help)) {}
    const std::string& name() const { return name_; }
    const std::string& help() const { return help_; }

    template <typename T>
    void value(const std::string& opt, T& target, const std::string& help, bool required = false) {
        Option o;
        o.name = opt;
        o.help = help;
        o.required = required;
        o.shown_default = show(target);
        o.set = [&target, opt](const std::string& v) { target = parse_number<T>(opt, v); };
        opts_.push_back(std::move(o));
    }
    void text(const std::string& opt, std::string& target, const std::string& help, bool required = false) {
        Option o;
        o.name = opt;
        o.help = help;
        o.required = required;
        o.shown_default = target;
        o.set = [&target](const std::string& v) { target = v; };
        opts_.push_back(std::move(o));
    }
    template <typename T>
    void list(const std::string& opt, std::vector<T>& target, const std::string& help) {
        Option o;
        o.name = opt;
        o.help = help;
        for (size_t i = 0; i < target.size(); ++i) o.shown_default += (i ? "," : "") + show(target[i]);
        o.set = [&target, opt](const std::string& v) {
            target.clear();
            for (const std::string& part : split_commas(v)) target.push_back(parse_number<T>(opt, part));
        };
        opts_.push_back(std::move(o));
    }
    void flag(const std::string& opt, bool& target, const std::string& help) {
        Option o;
        o.name = opt;
        o.help = help;
        o.flag = true;
        o.set = [&target](const std::string&) { target = true; };
        opts_.push_back(std::move(o));
    }

    // args: the words after the subcommand name
    void parse(const std::vector<std::string>& args) {
        for (size_t i = 0; i < args.size(); ++i) {
            std::string word = args[i];
            if (word == "--help" || word == "-h") throw HelpRequested{};
            std::string val;
            bool has_inline = false;
            const size_t eq = word.find('=');
            if (word.rfind("--", 0) == 0 && eq != std::string::npos) {
                val = word.substr(eq + 1);
                word = word.substr(0, eq);
                has_inline = true;
            }
            Option* o = find(word);
            if (!o) throw UsageError("unknown option for '" + name_ + "': " + word);
            if (o->flag) {
                if (has_inline) throw UsageError(word + " takes no value");
                o->set("");
            } else {
                if (!has_inline) {
                    if (i + 1 >= args.size()) throw UsageError(word + " needs a value");
                    val = args[++i];
                }
                o->set(val);
            }
            o->seen = true;
        }
        for (const Option& o : opts_)
            if (o.required && !o.seen) throw UsageError(o.name + " is required");
    }

    void print_help(const char* prog) const {
        std::printf("%s\nUsage: %s %s [OPTIONS]\n\nOptions:\n", help_.c_str(), prog, name_.c_str());
        for (const Option& o : opts_) {
            std::string left = o.name + (o.flag ? "" : " VALUE");
            std::printf("  %-28s %s", left.c_str(), o.help.c_str());
            if (o.required) std::printf(" (required)");
            if (!o.flag && !o.shown_default.empty()) std::printf(" [default: %s]", o.shown_default.c_str());
            std::printf("\n");
        }
    }

  private:
    Option* find(const std::string& n) {
        for (Option& o : opts_)
            if (o.name == n) return &o;
        return nullptr;
    }
    template <typename T>
    static std::string show(const T& v) {
        if constexpr (std::is_same_v<T, double>)
            return format_double(v);
        else
            return std::to_string(v);
    }

    std::string name_, help_;
    std::vector<Option> opts_;
};

// ------------------------------------------------------------------------- the subcommands
double mean_of(const std::vector<double>& values) {
    double sum = 0.0;
    for (double v : values) sum += v;
    return sum / static_cast<double>(values.size());
}

double sample_variance(const std::vector<double>& values) {  // unbiased; 0 below two samples
    if (values.size() < 2) return 0.0;
    const double m = mean_of(values);
    double sum = 0.0;
    for (double v : values) sum += (v - m) * (v - m);
    return sum / static_cast<double>(values.size() - 1);
}

// One file-backed instance for every run, or generator parameters, optionally re-seeded per run
// index (derive_seed(seed, run)) so that runs compared across settings see matched instances.
struct InstanceSource {
    std::string path;
    ffsga::GenParams gen;
    bool vary_per_run = false;
    ffsga::Instance fixed;

    void prepare() {
        if (!path.empty() && vary_per_run)
            throw ffsga::ConfigError("--vary-instance regenerates instances and cannot be combined with --instance");
        if (!path.empty())
            fixed = ffsga::load_instance(path);
        else if (!vary_per_run)
            fixed = ffsga::generate(gen);
    }
    ffsga::Instance for_run(int run) const {
        if (!vary_per_run) return fixed;
        ffsga::GenParams p = gen;
        p.seed = ffsga::derive_seed(gen.seed, static_cast<std::uint64_t>(run));
        return ffsga::generate(p);
    }
};

void generator_flags(Command& c, ffsga::GenParams& g, const char* seed_name) {
    c.value("--jobs", g.num_jobs, "number of jobs");
    c.value("--stages", g.num_stages, "number of stages");
    c.list("--machines", g.machines_per_stage, "machines per stage; one value is broadcast to every stage");
    c.value("--wt", g.weight, "tardiness weight in the objective");
    c.value(seed_name, g.seed, "instance generator seed");
    c.flag("--integer-times", g.integer_times, "round processing times to whole units");
}

void broadcast_machines(ffsga::GenParams& g) {
    if (g.machines_per_stage.size() == 1 && g.num_stages > 1)
        g.machines_per_stage.assign(static_cast<size_t>(g.num_stages), g.machines_per_stage[0]);
}

void run_flags(Command& c, ffsga::RunConfig& r) {
    c.value("--population", r.population, "total population size");
    c.value("--generations", r.generations, "generation budget");
    c.value("--gap", r.migration_gap, "generations between migration checks");
    c.value("--theta", r.theta, "migration threshold in [0, 1]");
    c.value("--seed", r.seed, "master GA seed");
    c.value("--workers", r.workers, "data-parallel workers per island (accepted; the GPU ignores it)");
    c.value("--cellular-crossover", r.cellular.crossover_rate, "cellular island crossover rate");
    c.value("--cellular-mutation", r.cellular.mutation_rate, "cellular island per-gene mutation rate");
    c.value("--pseudo-crossover", r.pseudo.crossover_rate, "pseudo island crossover rate");
    c.flag("--pseudo-fit-from-archive", r.pseudo_fit_from_archive,
           "feed the migration policy from the pseudo archive instead of the live population");
}

void source_flags(Command& c, InstanceSource& s) {
    c.text("--instance", s.path, "instance JSON path (omit to generate from the flags below)");
    generator_flags(c, s.gen, "--instance-seed");
    c.flag("--vary-instance", s.vary_per_run, "regenerate the instance for every run index");
}

void write_table(const std::string& csv, const std::string& out_path) {
    std::fputs(csv.c_str(), stdout);
    if (!out_path.empty()) {
        ffsga::write_text_file(out_path, csv);
        std::printf("wrote %s\n", out_path.c_str());
    }
}

int cmd_generate(const ffsga::GenParams& gen, const std::string& out_path) {
    ffsga::Instance inst = ffsga::generate(gen);
    ffsga::save_instance(inst, out_path);
    std::string machines;
    for (int m : inst.machines_per_stage) machines += (machines.empty() ? "" : " ") + std::to_string(m);
    auto [lo, hi] = std::minmax_element(inst.due.begin(), inst.due.end());
    std::printf("instance: %d jobs, %d stages, machines %s, weight %s\n", inst.num_jobs, inst.num_stages,
                machines.c_str(), format_double(inst.weight).c_str());
    std::printf("mean total load: %s\n", format_double(ffsga::mean_total_load(inst)).c_str());
    std::printf("due range: [%s, %s]\n", format_double(*lo).c_str(), format_double(*hi).c_str());
    std::printf("wrote %s\n", out_path.c_str());
    return 0;
}

int cmd_solve(const std::string& instance_path, ffsga::RunConfig cfg, const std::string& mode, bool serialized,
              const std::string& out_path, const std::string& trace_path) {
    cfg.mode = ffsga::parse_run_mode(mode);
    ffsga::Instance inst = ffsga::load_instance(instance_path);
    ffsga::RunResult res = serialized ? ffsga::run_serialized(cfg, inst) : ffsga::run(cfg, inst);
    ffsga::save_result_json(res, cfg, out_path);
    if (!trace_path.empty()) ffsga::save_trace_csv(res, trace_path);
    std::printf("best objective: %s (makespan %s, total tardiness %s)\n", format_double(res.best_objective).c_str(),
                format_double(res.best_makespan).c_str(), format_double(res.best_tardiness).c_str());
    std::printf("migrations executed: %zu\n", res.migrations.size());
    std::printf("total seconds: %s\n", format_double(res.timings.total_seconds).c_str());
    std::printf("wrote %s\n", out_path.c_str());
    if (!trace_path.empty()) std::printf("wrote %s\n", trace_path.c_str());
    return 0;
}

int cmd_sweep_gap(InstanceSource& src, ffsga::RunConfig cfg, const std::vector<int>& gaps, int runs,
                  const std::string& out_path) {
    if (gaps.empty()) throw ffsga::ConfigError("--gaps needs at least one value");
    if (runs < 1) throw ffsga::ConfigError("--runs must be at least 1");
    src.prepare();
    const std::uint64_t master = cfg.seed;
    std::string csv = "gap,mean_objective,std\n";
    for (int gap : gaps) {
        std::vector<double> obj;
        for (int r = 0; r < runs; ++r) {
            ffsga::RunConfig c = cfg;
            c.migration_gap = gap;
            c.seed = ffsga::derive_seed(master, static_cast<std::uint64_t>(r));
            obj.push_back(ffsga::run(c, src.for_run(r)).best_objective);
        }
        csv += std::to_string(gap) + "," + format_double(mean_of(obj)) + "," +
               format_double(std::sqrt(sample_variance(obj))) + "\n";
    }
    write_table(csv, out_path);
    return 0;
}

int cmd_compare(InstanceSource& src, ffsga::RunConfig cfg, int runs, const std::string& out_path) {
    if (runs < 2) throw ffsga::ConfigError("--runs must be at least 2 to report a variance");
    src.prepare();
    const std::uint64_t master = cfg.seed;
    struct Row {
        const char* label;
        ffsga::RunMode mode;
    };
    const Row rows[] = {{"Heterogeneous", ffsga::RunMode::dual},
                        {"Cellular", ffsga::RunMode::cellular_only},
                        {"Pseudo", ffsga::RunMode::pseudo_only}};
    std::string csv = "algorithm,best,average,variance\n";
    for (const Row& row : rows) {
        std::vector<double> obj;
        for (int r = 0; r < runs; ++r) {
            ffsga::RunConfig c = cfg;
            c.mode = row.mode;
            c.seed = ffsga::derive_seed(master, static_cast<std::uint64_t>(r));
            obj.push_back(ffsga::run(c, src.for_run(r)).best_objective);
        }
        csv += std::string(row.label) + "," + format_double(*std::min_element(obj.begin(), obj.end())) + "," +
               format_double(mean_of(obj)) + "," + format_double(sample_variance(obj)) + "\n";
    }
    write_table(csv, out_path);
    return 0;
}

int cmd_bench_time(InstanceSource& src, ffsga::RunConfig cfg, const std::vector<int>& pops,
                   const std::string& out_path) {
    if (pops.empty()) throw ffsga::ConfigError("--populations needs at least one value");
    src.prepare();
    std::string csv = "population,concurrent_seconds,serialized_seconds,speedup\n";
    for (int pop : pops) {
        ffsga::RunConfig c = cfg;
        c.population = pop;
        ffsga::Instance inst = src.for_run(0);
        ffsga::RunResult a = ffsga::run(c, inst);
        ffsga::RunResult b = ffsga::run_serialized(c, inst);
        if (a.best_objective != b.best_objective)
            throw ffsga::ContractError("concurrent and serialized runs disagree; determinism contract broken");
        csv += std::to_string(pop) + "," + format_double(a.timings.total_seconds) + "," +
               format_double(b.timings.total_seconds) + "," +
               format_double(b.timings.total_seconds / a.timings.total_seconds) + "\n";
    }
    write_table(csv, out_path);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    const char* prog = "ffsga";
    const char* about = "flexible flow shop solver (B200): dual heterogeneous island GA with adaptive migration";
    std::vector<std::string> args(argv + 1, argv + argc);

    int device = -1;  // --device is accepted anywhere
    for (size_t i = 0; i < args.size(); ++i) {
        if (args[i] == "--device" && i + 1 < args.size()) {
            try {
                device = parse_number<int>("--device", args[i + 1]);
            } catch (const std::exception& e) {
                std::fprintf(stderr, "error: %s\n", e.what());
                return 2;
            }
            args.erase(args.begin() + (long)i, args.begin() + (long)i + 2);
            break;
        }
    }
    if (device >= 0) setenv("FFSGA_DEVICE", std::to_string(device).c_str(), 1);

    ffsga::GenParams gen;
    std::string gen_out = "instance.json";
    Command generate("generate", "write a random instance file");
    generator_flags(generate, gen, "--seed");
    generate.text("--out", gen_out, "output instance path");

    ffsga::RunConfig solve_cfg;
    std::string solve_instance, solve_mode = "dual", solve_out = "result.json", solve_trace;
    bool solve_serialized = false;
    Command solve("solve", "run one GA configuration on an instance");
    solve.text("--instance", solve_instance, "instance JSON path", true);
    run_flags(solve, solve_cfg);
    solve.text("--mode", solve_mode, "dual | cellular | pseudo");
    solve.flag("--serialized", solve_serialized, "advance islands one after the other instead of concurrently");
    solve.text("--out", solve_out, "result JSON path");
    solve.text("--trace", solve_trace, "per-generation trace CSV path");

    InstanceSource sweep_src;
    ffsga::RunConfig sweep_cfg;
    std::vector<int> sweep_gaps = {10, 50, 100, 200, 400, 500, 800};
    int sweep_runs = 50;
    std::string sweep_out;
    Command sweep("sweep-gap", "mean final objective as a function of the migration gap");
    source_flags(sweep, sweep_src);
    run_flags(sweep, sweep_cfg);
    sweep.list("--gaps", sweep_gaps, "migration gaps to sweep");
    sweep.value("--runs", sweep_runs, "runs per gap value");
    sweep.text("--out", sweep_out, "also write the CSV here");

    InstanceSource cmp_src;
    ffsga::RunConfig cmp_cfg;
    int cmp_runs = 50;
    std::string cmp_out;
    Command compare("compare", "dual vs cellular-only vs pseudo-only quality with matched seeds");
    source_flags(compare, cmp_src);
    run_flags(compare, cmp_cfg);
    compare.value("--runs", cmp_runs, "runs per algorithm");
    compare.text("--out", cmp_out, "also write the CSV here");

    InstanceSource bench_src;
    ffsga::RunConfig bench_cfg;
    bench_cfg.generations = 200;  // desk-scale timing default (main.cpp:322)
    std::vector<int> bench_pops = {512, 1024, 2048, 4096};
    std::string bench_out;
    Command bench("bench-time", "concurrent vs serialized wall-clock across population sizes");
    source_flags(bench, bench_src);
    run_flags(bench, bench_cfg);
    bench.list("--populations", bench_pops, "population sizes to time");
    bench.text("--out", bench_out, "also write the CSV here");

    Command* commands[] = {&generate, &solve, &sweep, &compare, &bench};
    auto top_help = [&] {
        std::printf("%s\nUsage: %s [--device N] SUBCOMMAND [OPTIONS]\n\nSubcommands:\n", about, prog);
        for (Command* c : commands) std::printf("  %-12s %s\n", c->name().c_str(), c->help().c_str());
    };
    if (args.empty()) {
        std::fprintf(stderr, "error: a subcommand is required (generate, solve, sweep-gap, compare, bench-time)\n");
        return 2;
    }
    if (args[0] == "--help" || args[0] == "-h") {
        top_help();
        return 0;
    }
    Command* cmd = nullptr;
    for (Command* c : commands)
        if (c->name() == args[0]) cmd = c;
    if (!cmd) {
        std::fprintf(stderr, "error: unknown subcommand: %s\n", args[0].c_str());
        return 2;
    }
    try {
        cmd->parse(std::vector<std::string>(args.begin() + 1, args.end()));
    } catch (const HelpRequested&) {
        cmd->print_help(prog);
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
    try {
        if (cmd == &generate) {
            broadcast_machines(gen);
            return cmd_generate(gen, gen_out);
        }
        if (cmd == &solve)
            return cmd_solve(solve_instance, solve_cfg, solve_mode, solve_serialized, solve_out, solve_trace);
        if (cmd == &sweep) {
            broadcast_machines(sweep_src.gen);
            return cmd_sweep_gap(sweep_src, sweep_cfg, sweep_gaps, sweep_runs, sweep_out);
        }
        if (cmd == &compare) {
            broadcast_machines(cmp_src.gen);
            return cmd_compare(cmp_src, cmp_cfg, cmp_runs, cmp_out);
        }
        if (cmd == &bench) {
            broadcast_machines(bench_src.gen);
            return cmd_bench_time(bench_src, bench_cfg, bench_pops, bench_out);
        }
    } catch (const std::exception& e) {
        std::string msg = e.what();
        std::replace(msg.begin(), msg.end(), '\n', ' ');
        std::fprintf(stderr, "error: %s\n", msg.c_str());
        return 2;
    }
    return 2;
}
