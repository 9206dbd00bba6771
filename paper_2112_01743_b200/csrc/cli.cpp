// `chebpr` command-line front end, the same surface as the
// reference CLI (/root/reference/proj/tools/chebpr_main.cpp:63-249): subcommands gen / run /
// compare / coeffs, the same flags, CSV outputs (include/chebpr/csv.hpp) and exit codes
// (0 success, 1 usage / input / validation problem, 2 numeric failure, :239-248).
//
// B200 specifics (additive flags):
//  * `run` loads the file straight onto the device (GPU parse + K1 build, csrc/ingest.cu)
//    and solves on that resident handle through the C-ABI (cheb_cpaa / cheb_power): no
//    host CSR round trip.  --device N picks the GPU, --mode auto|fast|bitexact the schedule
//    (auto: bit-exact storage-order sums up to 2^20 CSR entries, the degree-binned FAST
//    kernel above; CHEBPR_MODE overrides auto), --precision 64|32 the vector type (cpaa).
//  * `gen` also writes the BASELINE config graphs: --model rmat (--scale, --edge-factor)
//    and --model chung-lu (--n, --gamma, --wmin, --wmax, --draws).
// CLI11 is not available here, so the parser is a small one of our own with CLI11's
// observable behaviour for these flags: `--opt value` or `--opt=value`, required options,
// member checks, mutually exclusive options, comma lists, unknown arguments rejected.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "chebpr/coefficients.hpp"
#include "chebpr/compare.hpp"
#include "chebpr/cpaa.hpp"
#include "chebpr/csv.hpp"
#include "chebpr/errors.hpp"
#include "chebpr/generate.hpp"
#include "chebpr/graph_io.hpp"
#include "chebpr/power.hpp"
#include "chebpr_cuda.h"

namespace {

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- argument parsing
struct Option {
    std::string name;  // "--input"
    std::string help;
    std::function<bool(const std::string&)> set;  // false: not convertible
    bool flag = false;
    bool list = false;  // comma / space separated values
    bool required = false;
    std::vector<std::string> members;  // allowed values (empty: any)
    std::vector<std::string> excludes;
    std::string dflt;
    bool seen = false;
};

template <class T>
bool convert(const std::string& s, T& out) {
    if (s.empty()) return false;
    char* end = nullptr;
    errno = 0;
    if constexpr (std::is_same_v<T, double>) {
        out = std::strtod(s.c_str(), &end);
    } else if constexpr (std::is_same_v<T, uint64_t>) {
        if (s[0] == '-') return false;
        out = std::strtoull(s.c_str(), &end, 10);
    } else {
        const long long v = std::strtoll(s.c_str(), &end, 10);
        out = (T)v;
        if ((long long)out != v) return false;
    }
    return errno == 0 && end && *end == '\0';
}

class Command {
public:
    Command(std::string name, std::string help) : name_(std::move(name)), help_(std::move(help)) {}
    const std::string& name() const { return name_; }
    const std::string& help() const { return help_; }

    template <class T>
    Option& option(const std::string& name, T& dst, const std::string& help) {
        Option o;
        o.name = name;
        o.help = help;
        o.set = [&dst](const std::string& v) { return convert(v, dst); };
        if constexpr (std::is_same_v<T, double>) {
            char b[40];
            std::snprintf(b, sizeof b, "%g", dst);
            o.dflt = b;
        } else {
            o.dflt = std::to_string(dst);
        }
        opts_.push_back(std::move(o));
        return opts_.back();
    }
    Option& option(const std::string& name, std::string& dst, const std::string& help) {
        Option o;
        o.name = name;
        o.help = help;
        o.set = [&dst](const std::string& v) {
            dst = v;
            return true;
        };
        o.dflt = dst;
        opts_.push_back(std::move(o));
        return opts_.back();
    }
    Option& list(const std::string& name, std::vector<int>& dst, const std::string& help) {
        Option o;
        o.name = name;
        o.help = help;
        o.list = true;
        auto first = std::make_shared<bool>(true);
        o.set = [&dst, first](const std::string& v) {
            if (*first) dst.clear();
            *first = false;
            int x = 0;
            if (!convert(v, x)) return false;
            dst.push_back(x);
            return true;
        };
        for (size_t i = 0; i < dst.size(); ++i) o.dflt += (i ? "," : "") + std::to_string(dst[i]);
        opts_.push_back(std::move(o));
        return opts_.back();
    }
    Option& flag(const std::string& name, bool& dst, const std::string& help) {
        Option o;
        o.name = name;
        o.help = help;
        o.flag = true;
        o.set = [&dst](const std::string& v) {
            if (v == "true" || v == "1" || v.empty()) dst = true;
            else if (v == "false" || v == "0") dst = false;
            else return false;
            return true;
        };
        opts_.push_back(std::move(o));
        return opts_.back();
    }

    // Parses argv[i..argc); throws UsageError with a CLI11-style message.
    void parse(int argc, char** argv, int i) {
        while (i < argc) {
            std::string tok = argv[i++];
            if (tok == "-h" || tok == "--help") {
                print_help(stdout);
                std::exit(0);
            }
            if (tok.rfind("--", 0) != 0)
                throw UsageError("The following argument was not expected: " + tok);
            std::string key = tok, val;
            bool inline_val = false;
            const size_t eq = tok.find('=');
            if (eq != std::string::npos) {
                key = tok.substr(0, eq);
                val = tok.substr(eq + 1);
                inline_val = true;
            }
            Option* o = find(key);
            if (!o) throw UsageError("The following argument was not expected: " + tok);
            o->seen = true;
            if (o->flag) {
                if (!o->set(inline_val ? val : std::string()))
                    throw UsageError(key + ": could not convert '" + val + "' to a flag value");
                continue;
            }
            std::vector<std::string> vals;
            if (inline_val) {
                vals.push_back(val);
            } else {
                if (i >= argc || std::string(argv[i]).rfind("--", 0) == 0)
                    throw UsageError(key + " requires an argument");
                vals.push_back(argv[i++]);
                while (o->list && i < argc && std::string(argv[i]).rfind("--", 0) != 0) vals.push_back(argv[i++]);
            }
            for (const std::string& v0 : vals) {
                std::vector<std::string> parts;
                if (o->list) {
                    size_t a = 0;
                    while (true) {
                        const size_t b = v0.find(',', a);
                        parts.push_back(v0.substr(a, b == std::string::npos ? std::string::npos : b - a));
                        if (b == std::string::npos) break;
                        a = b + 1;
                    }
                } else {
                    parts.push_back(v0);
                }
                for (const std::string& v : parts) {
                    if (!o->members.empty()) {
                        bool ok = false;
                        for (const auto& m : o->members) ok = ok || m == v;
                        if (!ok) throw UsageError(key + ": " + v + " not in {" + join(o->members) + "}");
                    }
                    if (!o->set(v)) throw UsageError(key + ": Could not convert: " + v);
                }
            }
        }
        for (const Option& o : opts_) {
            if (o.required && !o.seen) throw UsageError(o.name + " is required");
            if (!o.seen) continue;
            for (const std::string& x : o.excludes) {
                const Option* other = find_c(x);
                if (other && other->seen) throw UsageError(o.name + " excludes " + x);
            }
        }
    }

    void print_help(std::FILE* f) const {
        std::fprintf(f, "%s\nUsage: chebpr %s [OPTIONS]\n\nOptions:\n", help_.c_str(), name_.c_str());
        for (const Option& o : opts_) {
            std::string l = "  " + o.name + (o.flag ? "" : (o.list ? " INT,..." : " VALUE"));
            std::fprintf(f, "%-28s %s", l.c_str(), o.help.c_str());
            if (!o.members.empty()) std::fprintf(f, " {%s}", join(o.members).c_str());
            if (o.required) std::fprintf(f, " (required)");
            else if (!o.flag && !o.dflt.empty()) std::fprintf(f, " [%s]", o.dflt.c_str());
            std::fputc('\n', f);
        }
    }

    bool seen(const std::string& name) const {
        const Option* o = find_c(name);
        return o && o->seen;
    }

private:
    static std::string join(const std::vector<std::string>& v) {
        std::string s;
        for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + v[i];
        return s;
    }
    Option* find(const std::string& k) {
        for (auto& o : opts_)
            if (o.name == k) return &o;
        return nullptr;
    }
    const Option* find_c(const std::string& k) const {
        for (auto& o : opts_)
            if (o.name == k) return &o;
        return nullptr;
    }
    std::string name_, help_;
    std::vector<Option> opts_;
};

// ---------------------------------------------------------------- helpers
struct LoadFlags {
    std::string input;
    std::string format = "edgelist";
    bool drop_isolated = false, symmetrize = false, dedup = true, keep_multi = false;
    int device = 0;
};

void add_load_flags(Command& c, LoadFlags& lf, bool device) {
    c.option("--input", lf.input, "graph file to load").required = true;
    c.option("--format", lf.format, "input format").members = {"edgelist", "mtx"};
    c.flag("--drop-isolated", lf.drop_isolated, "drop zero-degree vertices (renumbers the rest) instead of failing");
    c.flag("--symmetrize", lf.symmetrize, "treat a general Matrix Market file as undirected even if one-sided");
    c.flag("--dedup", lf.dedup, "collapse duplicate edges (default)");
    c.flag("--keep-multi", lf.keep_multi, "keep duplicate edges as multiplicity instead of collapsing")
        .excludes = {"--dedup"};
    if (device) c.option("--device", lf.device, "CUDA device ordinal");
}

// C-ABI status -> the reference's exception type (message from cheb_last_error()).
void check(cheb_status s) {
    if (s == CHEB_OK) return;
    const std::string m = cheb_last_error();
    switch (s) {
        case CHEB_VALIDATION: throw chebpr::ValidationError(m);
        case CHEB_DOMAIN: throw chebpr::DomainError(m);
        case CHEB_NUMERIC: throw chebpr::NumericError(m);
        case CHEB_INVALID_ARG: throw std::invalid_argument(m);
        case CHEB_CAPACITY: throw chebpr::CapacityError(m);
        case CHEB_PARSE: throw chebpr::ParseError(m);
        default: throw chebpr::Error(m);
    }
}

// The graph resident on the device (GPU parse + K1), with the loader's stats.
struct DeviceFile {
    cheb_graph_t h = nullptr;
    cheb_graph_stats st{};
    explicit DeviceFile(const LoadFlags& lf) {
        cheb_load_opts o;
        cheb_load_opts_default(&o);
        o.dedup = lf.keep_multi ? 0 : 1;
        o.drop_isolated = lf.drop_isolated ? 1 : 0;
        o.symmetrize = lf.symmetrize ? 1 : 0;
        o.device = lf.device;
        check(lf.format == "mtx" ? cheb_graph_load_matrix_market(lf.input.c_str(), &o, &h, &st)
                                 : cheb_graph_load_edge_list(lf.input.c_str(), &o, &h, &st));
        // finish()'s warnings (graph_io.cpp:38-40, 134-138)
        if (st.weights_ignored)
            std::fprintf(stderr, "warning: %s: real weights ignored, using pattern only\n", lf.input.c_str());
        if (st.isolated_dropped > 0)
            std::fprintf(stderr, "warning: dropped %lld isolated vertices\n", (long long)st.isolated_dropped);
    }
    ~DeviceFile() { cheb_graph_free(h); }
    DeviceFile(const DeviceFile&) = delete;
    DeviceFile& operator=(const DeviceFile&) = delete;
};

chebpr::LoadedGraph load_host(const LoadFlags& lf) {
    chebpr::LoadOptions o;
    o.dedup = !lf.keep_multi;
    o.drop_isolated = lf.drop_isolated;
    o.symmetrize = lf.symmetrize;
    return lf.format == "mtx" ? chebpr::load_matrix_market(lf.input, o) : chebpr::load_edge_list(lf.input, o);
}

int mode_of(const std::string& m, int64_t nnz) {
    std::string s = m;
    if (s == "auto") {
        const char* env = std::getenv("CHEBPR_MODE");
        if (env && (std::strcmp(env, "fast") == 0 || std::strcmp(env, "bitexact") == 0)) s = env;
    }
    if (s == "fast") return CHEB_MODE_FAST;
    if (s == "bitexact") return CHEB_MODE_BITEXACT;
    return nnz <= chebpr::kAutoExactNnz ? CHEB_MODE_BITEXACT : CHEB_MODE_FAST;
}

std::vector<chebpr::TraceRow> rows_of(const std::vector<cheb_trace_row>& t, int rounds) {
    std::vector<chebpr::TraceRow> out((size_t)std::max(rounds, 0));
    for (int i = 0; i < rounds; ++i) {
        auto& r = out[(size_t)i];
        r.k = t[(size_t)i].k;
        r.c_k = t[(size_t)i].c_k;
        r.S_k = t[(size_t)i].S_k;
        r.residual_mass = t[(size_t)i].residual_mass;
        r.l1_change = t[(size_t)i].l1_change;
        r.elapsed_ms = t[(size_t)i].elapsed_ms;
        r.mass_T = t[(size_t)i].mass_T;
        r.err = t[(size_t)i].err;
        r.err_l1 = t[(size_t)i].err_l1;
    }
    return out;
}

void print_usage(std::FILE* f, const std::vector<Command*>& cmds) {
    std::fprintf(f, "Chebyshev-accelerated PageRank for undirected graphs (B200)\n"
                    "Usage: chebpr SUBCOMMAND [OPTIONS]\n\nSubcommands:\n");
    for (const Command* c : cmds) std::fprintf(f, "  %-10s %s\n", c->name().c_str(), c->help().c_str());
}

}  // namespace

int main(int argc, char** argv) {
    // gen
    Command gen("gen", "generate a synthetic graph as an edge list");
    std::string gen_model, gen_output;
    int64_t gen_n = 0, gen_k = 0, gen_ef = 16, gen_draws = -1;
    int gen_scale = 0;
    double gen_p = -1.0, gen_avg_deg = -1.0, gen_gamma = 2.1, gen_wmin = 2.0, gen_wmax = 50000.0;
    uint64_t gen_seed = 1;
    {
        Option& o = gen.option("--model", gen_model, "graph model");
        o.members = {"ring", "star", "regular", "gnp", "rmat", "chung-lu"};
        o.required = true;
    }
    gen.option("--n", gen_n, "vertex count (rmat: 2^scale)");
    gen.option("--k", gen_k, "degree (regular model)");
    gen.option("--p", gen_p, "edge probability (gnp model)");
    gen.option("--avg-deg", gen_avg_deg, "expected vertex degree (gnp model), p = avg/(n-1)").excludes = {"--p"};
    gen.option("--seed", gen_seed, "RNG seed (gnp, rmat, chung-lu)");
    gen.option("--scale", gen_scale, "log2 vertex count (rmat model)");
    gen.option("--edge-factor", gen_ef, "edges drawn per vertex (rmat model)");
    gen.option("--gamma", gen_gamma, "power-law exponent (chung-lu model)");
    gen.option("--wmin", gen_wmin, "smallest expected degree (chung-lu model)");
    gen.option("--wmax", gen_wmax, "largest expected degree (chung-lu model)");
    gen.option("--draws", gen_draws, "endpoint pairs drawn (chung-lu model; default 10 n)");
    gen.option("--output", gen_output, "edge-list file to write").required = true;

    // run
    Command run("run", "run one solver and write ranks (and a trace)");
    LoadFlags run_load;
    add_load_flags(run, run_load, true);
    std::string run_algo, run_output, run_trace, run_mode = "auto";
    double run_c = 0.85, run_eps = -1.0;
    int run_rounds = -1, run_parallelism = 1, run_max_rounds = 60, run_precision = 64;
    {
        Option& o = run.option("--algo", run_algo, "algorithm");
        o.members = {"cpaa", "power"};
        o.required = true;
    }
    run.option("--c", run_c, "damping factor");
    run.option("--eps", run_eps, "target error (resolved to a round count)");
    run.option("--rounds", run_rounds, "fixed round count").excludes = {"--eps"};
    run.option("--parallelism", run_parallelism, "worker count (accepted; results never depend on it)");
    run.option("--max-rounds", run_max_rounds, "round cap / budget");
    run.option("--output", run_output, "ranks CSV path");
    run.option("--trace", run_trace, "per-round trace CSV path");
    run.option("--mode", run_mode, "schedule").members = {"auto", "fast", "bitexact"};
    run.option("--precision", run_precision, "vector precision of the cpaa solve").members = {"64", "32"};

    // compare
    Command cmp("compare", "rounds-to-error comparison of both algorithms");
    LoadFlags cmp_load;
    add_load_flags(cmp, cmp_load, false);
    std::string cmp_output;
    double cmp_c = 0.85, cmp_eps = 1e-3;
    std::vector<int> cmp_parallelism = {1};
    int cmp_max_rounds = 60;
    cmp.option("--c", cmp_c, "damping factor");
    cmp.option("--eps", cmp_eps, "target max relative error");
    cmp.list("--parallelism", cmp_parallelism, "worker counts to sweep");
    cmp.option("--max-rounds", cmp_max_rounds, "round budget for the cpaa crossing search");
    cmp.option("--output", cmp_output, "comparison CSV path (stdout if omitted)");

    // coeffs
    Command coef("coeffs", "dump the coefficient table as CSV");
    std::string coef_output;
    double coef_c = 0.85, coef_tol = 1e-10;
    int coef_max_k = 60;
    bool coef_quad = false;
    coef.option("--c", coef_c, "damping factor");
    coef.option("--max-k", coef_max_k, "largest k");
    coef.flag("--quadrature-check", coef_quad, "add a quadrature column and report the max deviation");
    coef.option("--quad-tol", coef_tol, "quadrature tolerance");
    coef.option("--output", coef_output, "CSV path (stdout if omitted)");

    std::vector<Command*> cmds = {&gen, &run, &cmp, &coef};
    Command* sel = nullptr;
    try {
        if (argc < 2) throw UsageError("A subcommand is required");
        const std::string sub = argv[1];
        if (sub == "-h" || sub == "--help") {
            print_usage(stdout, cmds);
            return 0;
        }
        for (Command* c : cmds)
            if (c->name() == sub) sel = c;
        if (!sel) throw UsageError("The following argument was not expected: " + sub);
        sel->parse(argc, argv, 2);
        if (sel == &gen && gen_model != "rmat" && !gen.seen("--n")) throw UsageError("--n is required");
        if (sel == &gen && gen_model == "rmat" && !gen.seen("--scale")) throw UsageError("--scale is required");
    } catch (const UsageError& e) {
        std::fprintf(stderr, "%s\nRun with --help for more information.\n", e.what());
        return 1;
    }

    try {
        if (sel == &gen) {
            chebpr::EdgeList edges;
            std::string note = "chebpr gen model=" + gen_model;
            if (gen_model == "gnp") {
                if (gen_p < 0.0 && gen_avg_deg < 0.0) throw chebpr::DomainError("gnp needs --p or --avg-deg");
                const double p = gen_p >= 0.0 ? gen_p : gen_avg_deg / static_cast<double>(gen_n - 1);
                edges = chebpr::gnp_edges(gen_n, p, gen_seed);
                note += " n=" + std::to_string(gen_n) + " p=" + chebpr::fmt17(p) + " seed=" + std::to_string(gen_seed);
            } else if (gen_model == "ring") {
                edges = chebpr::ring_edges(gen_n);
                note += " n=" + std::to_string(gen_n);
            } else if (gen_model == "star") {
                edges = chebpr::star_edges(gen_n);
                note += " n=" + std::to_string(gen_n);
            } else if (gen_model == "regular") {
                if (gen_k < 1) throw chebpr::DomainError("regular needs --k >= 1");
                edges = chebpr::regular_edges(gen_n, gen_k);
                note += " n=" + std::to_string(gen_n) + " k=" + std::to_string(gen_k);
            } else if (gen_model == "rmat") {
                edges = chebpr::rmat_edges(gen_scale, gen_ef, 0.57, 0.19, 0.19, gen_seed);
                note += " scale=" + std::to_string(gen_scale) + " edge_factor=" + std::to_string(gen_ef) +
                        " a=0.57 b=0.19 c=0.19 seed=" + std::to_string(gen_seed);
            } else {
                const int64_t draws = gen_draws >= 0 ? gen_draws : 10 * gen_n;
                edges = chebpr::chung_lu_edges(gen_n, gen_gamma, gen_wmin, gen_wmax, draws, gen_seed);
                note += " n=" + std::to_string(gen_n) + " gamma=" + chebpr::fmt17(gen_gamma) + " wmin=" +
                        chebpr::fmt17(gen_wmin) + " wmax=" + chebpr::fmt17(gen_wmax) + " draws=" +
                        std::to_string(draws) + " seed=" + std::to_string(gen_seed);
            }
            chebpr::write_edge_list(gen_output, edges, note);
            std::printf("wrote %s\n", gen_output.c_str());
        } else if (sel == &run) {
            if (run_eps <= 0.0 && run_rounds < 0) throw chebpr::DomainError("set one of --eps or --rounds");
            DeviceFile df(run_load);
            cheb_graph_info info;
            check(cheb_graph_get_info(df.h, &info));
            const int64_t n = info.n;
            // bit-exact sums are fp64 only: auto picks FAST for an fp32 solve
            const int mode = run_precision == 32 && run_mode == "auto" ? CHEB_MODE_FAST : mode_of(run_mode, info.nnz);
            chebpr::Vector ranks(n);
            std::vector<cheb_trace_row> tr;
            int rounds = 0;
            double total = 0.0;
            if (run_algo == "cpaa") {
                cheb_cpaa_opts o;
                cheb_cpaa_opts_default(&o);
                o.c = run_c;
                o.rounds = run_rounds;
                o.eps = run_eps;
                o.max_rounds = run_max_rounds;
                o.parallelism = run_parallelism;
                o.mode = mode;
                o.precision = run_precision;
                tr.resize((size_t)std::max(run_max_rounds, 0) + 1);
                check(cheb_cpaa(df.h, &o, nullptr, 0, ranks.data(), tr.data(), &rounds, &total));
                if (!run_trace.empty()) chebpr::write_cpaa_trace_csv(run_trace, rows_of(tr, rounds), false);
            } else {
                cheb_power_opts o;
                cheb_power_opts_default(&o);
                o.c = run_c;
                o.rounds = run_rounds;
                o.tol = run_eps;
                o.max_rounds = run_max_rounds;
                o.parallelism = run_parallelism;
                o.mode = mode;
                const int cap = std::max(run_rounds >= 0 ? run_rounds : run_max_rounds, 0) + 1;
                tr.resize((size_t)cap);
                check(cheb_power(df.h, &o, nullptr, 0, ranks.data(), tr.data(), cap, &rounds, &total));
                if (!run_trace.empty()) chebpr::write_power_trace_csv(run_trace, rows_of(tr, rounds), false);
            }
            if (!run_output.empty()) chebpr::write_ranks_csv(run_output, ranks);
            double ms = 0.0;
            for (int i = 0; i < rounds; ++i) ms += tr[(size_t)i].elapsed_ms;
            std::printf("n=%lld m=%lld algo=%s rounds=%d elapsed_ms=%.3f\n", (long long)df.st.n,
                        (long long)df.st.m, run_algo.c_str(), rounds, ms);
        } else if (sel == &cmp) {
            chebpr::LoadedGraph lg = load_host(cmp_load);
            chebpr::CompareOptions o;
            o.c = cmp_c;
            o.eps = cmp_eps;
            o.parallelism = cmp_parallelism;
            o.cpaa_budget = cmp_max_rounds;
            std::fprintf(stderr, "comparing on n=%lld m=%lld (210-round reference)\n", (long long)lg.stats.n,
                         (long long)lg.stats.m);
            const auto rows = chebpr::compare_algorithms(lg.graph, o);
            if (cmp_output.empty()) chebpr::write_compare_csv(stdout, rows);
            else chebpr::write_compare_csv(cmp_output, rows);
        } else {
            const chebpr::CoefficientTable table = chebpr::coefficients(coef_c, coef_max_k);
            chebpr::CoefficientTable quad;
            if (coef_quad) quad = chebpr::coefficients_quadrature(coef_c, coef_max_k, coef_tol);
            std::FILE* out = stdout;
            if (!coef_output.empty()) {
                out = std::fopen(coef_output.c_str(), "wb");
                if (!out) throw chebpr::ParseError("cannot write " + coef_output);
            }
            std::string text = coef_quad ? "k,c_k,err_bound_k,c_k_quadrature\n" : "k,c_k,err_bound_k\n";
            double worst = 0.0;
            for (int k = 0; k <= coef_max_k; ++k) {
                text += std::to_string(k) + "," + chebpr::fmt17(table.coeffs[(size_t)k]) + "," +
                        chebpr::fmt17(chebpr::err_bound(coef_c, k));
                if (coef_quad) {
                    worst = std::max(worst, std::abs(table.coeffs[(size_t)k] - quad.coeffs[(size_t)k]));
                    text += "," + chebpr::fmt17(quad.coeffs[(size_t)k]);
                }
                text += "\n";
            }
            std::fwrite(text.data(), 1, text.size(), out);
            if (out != stdout && std::fclose(out) != 0) throw chebpr::ParseError("write failed for " + coef_output);
            if (coef_quad)
                std::fprintf(stderr, "max closed-form vs quadrature deviation: %s\n", chebpr::fmt17(worst).c_str());
        }
        return 0;
    } catch (const chebpr::NumericError& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
