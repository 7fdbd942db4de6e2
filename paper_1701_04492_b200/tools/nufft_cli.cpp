// nufft — the command-line front end of the reference (proj/tools/nufft_main.cpp,
// nufft_app.hpp) on the B200 library: the same four subcommands, options, CSV
// files (include/nufft/csv.hpp) and exit codes, every transform on the GPU
// through the drop-in headers.
//
//   nufft transform --type {1|2|3|2d2|inv1|inv2} --in FILE... --out FILE
//                   [--eps E] [--tol T] [--threads N] [--seed S] [--fft]
//   nufft verify    [--n N...] [--gamma G...] [--eps E...] [--trials T] [--seed S] [--decay] --out FILE
//   nufft bench     [--n N...] [--eps E...] [--gamma G] [--trials T] [--seed S] --out FILE
//   nufft cgstudy   [--n N...] [--gamma G...] [--tol T] [--eps E] [--trials T] [--seed S] --out FILE
//
// Exit codes (nufft_app.hpp:6): 0 success, 1 verification failure, 2 I/O or
// usage, 3 domain (including a stalled CG and invalid numeric arguments).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "nufft/csv.hpp"
#include "nufft/nufft.hpp"
#include "nufft/oracle.hpp"
#include "nufft/random.hpp"

namespace {

constexpr int kOk = 0, kVerifyFail = 1, kIo = 2, kDomain = 3;

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- arguments
// --name value... : every value up to the next "--" token belongs to the option
struct Args {
    std::map<std::string, std::vector<std::string>> opt;
    bool has(const std::string& k) const { return opt.count(k) > 0; }
    const std::vector<std::string>& list(const std::string& k) const {
        static const std::vector<std::string> none;
        auto it = opt.find(k);
        return it == opt.end() ? none : it->second;
    }
    std::string one(const std::string& k) const {
        const auto& v = list(k);
        if (v.size() != 1) throw Usage("--" + k + " needs exactly one value");
        return v[0];
    }
};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& known,
           const std::vector<std::string>& flags) {
    Args a;
    std::string cur;
    for (int i = first; i < argc; ++i) {
        const std::string t = argv[i];
        if (t.size() > 2 && t[0] == '-' && t[1] == '-') {
            cur = t.substr(2);
            if (std::find(known.begin(), known.end(), cur) == known.end() &&
                std::find(flags.begin(), flags.end(), cur) == flags.end())
                throw Usage("unknown option " + t);
            a.opt[cur];
            if (std::find(flags.begin(), flags.end(), cur) != flags.end()) cur.clear();
        } else {
            if (cur.empty()) throw Usage("unexpected argument '" + t + "'");
            a.opt[cur].push_back(t);
        }
    }
    return a;
}

double to_double(const std::string& s, const char* what) {
    char* e = nullptr;
    const double v = std::strtod(s.c_str(), &e);
    if (e == s.c_str() || *e != '\0') throw Usage(std::string("bad ") + what + " '" + s + "'");
    return v;
}
unsigned long long to_u64(const std::string& s, const char* what) {
    char* e = nullptr;
    const unsigned long long v = std::strtoull(s.c_str(), &e, 10);
    if (e == s.c_str() || *e != '\0') throw Usage(std::string("bad ") + what + " '" + s + "'");
    return v;
}
template <class T, class F>
std::vector<T> values(const Args& a, const std::string& k, std::vector<T> dflt, F conv) {
    if (!a.has(k)) return dflt;
    std::vector<T> out;
    for (const auto& s : a.list(k)) out.push_back(conv(s));
    if (out.empty()) throw Usage("--" + k + " needs at least one value");
    return out;
}

// ---------------------------------------------------------------- timing
double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// median seconds of one call (nufft_app.hpp:36-55): one warm-up, the inner loop
// doubled until a measurement spans >= 2 ms, then `reps` measurements
template <class Fn>
double time_median(Fn&& fn, unsigned reps) {
    fn();
    std::size_t loops = 1;
    for (;;) {
        const double t0 = now();
        for (std::size_t i = 0; i < loops; ++i) fn();
        if (now() - t0 >= 2e-3 || loops >= (std::size_t(1) << 20)) break;
        loops *= 2;
    }
    std::vector<double> t(std::max(1u, reps));
    for (auto& v : t) {
        const double t0 = now();
        for (std::size_t i = 0; i < loops; ++i) fn();
        v = (now() - t0) / static_cast<double>(loops);
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

double norm2(const nufft::ComplexVector& v) {
    long double s = 0;
    for (const auto& z : v) s += std::norm(z);
    return static_cast<double>(std::sqrt(s));
}

// ---------------------------------------------------------------- transform
int cmd_transform(const Args& a) {
    const std::string type = a.one("type");
    const auto& in = a.list("in");
    const std::string out = a.one("out");
    if (in.empty()) throw Usage("--in needs input files");
    const double eps = a.has("eps") ? to_double(a.one("eps"), "--eps") : 2.2e-16;
    const double tol = a.has("tol") ? to_double(a.one("tol"), "--tol") : 1e-12;
    const unsigned threads = a.has("threads") ? (unsigned)to_u64(a.one("threads"), "--threads") : 1u;
    const bool plain = a.has("fft");
    auto need = [&](std::size_t k, const char* files) {
        if (in.size() != k) throw Usage("--type " + type + " needs --in " + files);
    };
    const double t_read = now();
    if (type == "2" || type == "inv2" || type == "1" || type == "inv1") {
        const bool two = type == "2" || type == "inv2";
        need(2, two ? "SAMPLES.csv DATA.csv" : "FREQS.csv DATA.csv");
        const auto pts = two ? nufft::read_samples(in[0]) : nufft::read_frequencies(in[0]);
        const auto data = nufft::read_complex_vector(in[1]);
        const bool forward = type == "2" || type == "1";
        if (plain) {  // the FFT baseline path of the reference CLI
            nufft::write_complex_vector(out, forward ? nufft::fft_forward(data) : nufft::fft_inverse(data));
            std::fprintf(stderr, "plain fft path, N=%zu\n", data.size());
            return kOk;
        }
        const double t_plan = now();
        nufft::ComplexVector result;
        std::size_t iters = 0, size = 0, rank = 0;
        double gamma = 0, t_exec = 0;
        auto finish_cg = [&](const nufft::CgReport& rep) {
            if (!rep.converged) {
                std::fprintf(stderr, "%s: cg stalled at residual %.3e after %zu iterations\n", type.c_str(),
                             rep.relativeResidual, rep.iterations);
                return false;
            }
            result = rep.solution;
            iters = rep.iterations;
            return true;
        };
        if (two) {
            const nufft::Plan2 plan = nufft::plan_nufft2(pts, eps);
            t_exec = now();
            size = plan.size(), rank = plan.rank(), gamma = plan.gamma();
            if (forward) result = nufft::exec_nufft2(plan, data, threads);
            else if (!finish_cg(nufft::inufft2(plan, data, tol))) return kDomain;
        } else {
            const nufft::Plan1 plan = nufft::plan_nufft1(pts, eps);
            t_exec = now();
            size = plan.size(), rank = plan.rank(), gamma = plan.gamma();
            if (forward) result = nufft::exec_nufft1(plan, data);
            else if (!finish_cg(nufft::inufft1(plan, data, tol))) return kDomain;
        }
        const double t_done = now();
        nufft::write_complex_vector(out, result);
        std::fprintf(stderr, "type=%s N=%zu K=%zu gamma=%.6g plan_s=%.6f online_s=%.6f", type.c_str(), size, rank,
                     gamma, t_exec - t_plan, t_done - t_exec);
        if (iters > 0) std::fprintf(stderr, " cg_iterations=%zu", iters);
        if (two) std::fprintf(stderr, " read_s=%.6f", t_plan - t_read);
        std::fprintf(stderr, "\n");
        return kOk;
    }
    if (type == "3") {
        need(3, "SAMPLES.csv FREQS.csv COEFFS.csv");
        const auto x = nufft::read_samples(in[0]);
        const auto w = nufft::read_frequencies(in[1]);
        const auto c = nufft::read_complex_vector(in[2]);
        const double t_plan = now();
        const nufft::Plan3 plan = nufft::plan_nufft3(x, w, eps);
        const double t_exec = now();
        const auto f = nufft::exec_nufft3(plan, c);
        const double t_done = now();
        nufft::write_complex_vector(out, f);
        std::fprintf(stderr, "type=3 N=%zu K=%zu effective_rank=%zu gamma=%.6g wraparound=%s plan_s=%.6f online_s=%.6f\n",
                     plan.size(), plan.factorsA.rank, plan.effective_rank(), plan.samples.gamma,
                     plan.bTrivial ? "none" : "rank2", t_exec - t_plan, t_done - t_exec);
        return kOk;
    }
    if (type == "2d2") {
        need(2, "SAMPLES2D.csv MATRIX.csv");
        std::vector<double> x, y;
        nufft::read_samples_2d(in[0], x, y);
        const nufft::ComplexMatrix C = nufft::read_complex_matrix(in[1]);
        const double t_plan = now();
        const nufft::Plan2D plan = nufft::plan_nufft2d2(x, y, C.rows, C.cols, eps);
        const double t_exec = now();
        const auto f = nufft::exec_nufft2d2(plan, C);
        const double t_done = now();
        nufft::write_complex_vector(out, f);
        std::fprintf(stderr, "type=2d2 N=%zu m=%zu n=%zu K1=%zu K2=%zu gammaX=%.6g gammaY=%.6g plan_s=%.6f online_s=%.6f\n",
                     plan.size(), plan.m, plan.n, plan.rank_x(), plan.rank_y(), plan.grid.gammaX, plan.grid.gammaY,
                     t_exec - t_plan, t_done - t_exec);
        return kOk;
    }
    throw Usage("unknown --type '" + type + "' (use 1, 2, 3, 2d2, inv1, inv2)");
}

// ---------------------------------------------------------------- verify
std::ofstream open_out(const std::string& path, const char* cmd) {
    std::ofstream f(path);
    if (!f) throw nufft::CsvError(path, 0, std::string(cmd) + ": cannot open for writing");
    return f;
}

int cmd_verify(const Args& a) {
    const auto ns = values<std::size_t>(a, "n", {64, 256}, [](const std::string& s) { return (std::size_t)to_u64(s, "--n"); });
    const auto gs = values<double>(a, "gamma", {0.0, 1.0 / 32, 1.0 / 8, 1.0 / 2}, [](const std::string& s) { return to_double(s, "--gamma"); });
    const auto es = values<double>(a, "eps", {2.2e-16, 1.2e-7, 9.8e-4}, [](const std::string& s) { return to_double(s, "--eps"); });
    const unsigned trials = a.has("trials") ? (unsigned)to_u64(a.one("trials"), "--trials") : 1u;
    const std::uint64_t seed = a.has("seed") ? to_u64(a.one("seed"), "--seed") : 1u;
    const bool decay = a.has("decay");
    auto csv = open_out(a.one("out"), "verify");
    csv << "N,gamma,eps,K,rel_error,bound,pass\n";
    nufft::GaussianSampler rng(seed);
    bool all = true;
    for (std::size_t n : ns)
        for (double g : gs) {
            const auto x = nufft::worst_grid(n, g);
            std::vector<double> w(n);
            for (std::size_t k = 0; k < n; ++k) w[k] = static_cast<double>(k);
            for (double eps : es) {
                const nufft::Plan2 plan = nufft::plan_nufft2(x, eps);
                for (unsigned t = 0; t < trials; ++t) {
                    nufft::ComplexVector c = rng.complex_vector(n);
                    if (decay)
                        for (std::size_t k = 0; k < n; ++k) c[k] /= static_cast<double>((k + 1) * (k + 1));
                    const auto fast = nufft::exec_nufft2(plan, c);
                    const auto exact = nufft::nudft_direct(x, w, c);
                    long double d = 0;
                    for (std::size_t j = 0; j < n; ++j) d += std::norm(fast[j] - exact[j]);
                    const double rel = static_cast<double>(std::sqrt(d)) / norm2(c);
                    const double bound = static_cast<double>(n) * eps;
                    const bool pass = rel <= bound;
                    all = all && pass;
                    char line[192];
                    std::snprintf(line, sizeof line, "%zu,%.17g,%.17g,%zu,%.9e,%.9e,%d\n", n, g, eps, plan.rank(), rel,
                                  bound, pass ? 1 : 0);
                    csv << line;
                }
            }
        }
    return all ? kOk : kVerifyFail;
}

// ---------------------------------------------------------------- bench
int cmd_bench(const Args& a) {
    const auto ns = values<std::size_t>(a, "n", {1024, 4096, 16384}, [](const std::string& s) { return (std::size_t)to_u64(s, "--n"); });
    const auto es = values<double>(a, "eps", {2.2e-16}, [](const std::string& s) { return to_double(s, "--eps"); });
    const double gamma = a.has("gamma") ? to_double(a.one("gamma"), "--gamma") : 0.5;
    const unsigned reps = a.has("trials") ? (unsigned)to_u64(a.one("trials"), "--trials") : 3u;
    const std::uint64_t seed = a.has("seed") ? to_u64(a.one("seed"), "--seed") : 1u;
    auto csv = open_out(a.one("out"), "bench");
    csv << "N,eps,K,plan_seconds,exec_seconds,fft_seconds_baseline,exec_over_fft_ratio\n";
    nufft::GaussianSampler rng(seed);
    for (std::size_t n : ns) {
        const auto x = nufft::worst_grid(n, gamma);
        const auto c = rng.complex_vector(n);
        for (double eps : es) {
            const double plan_s = time_median([&] { (void)nufft::plan_nufft2(x, eps); }, reps);
            const nufft::Plan2 plan = nufft::plan_nufft2(x, eps);
            const double exec_s = time_median([&] { (void)nufft::exec_nufft2(plan, c); }, reps);
            const double fft_s = time_median([&] { (void)nufft::fft_forward(c); }, reps);
            char line[224];
            std::snprintf(line, sizeof line, "%zu,%.17g,%zu,%.6e,%.6e,%.6e,%.3f\n", n, eps, plan.rank(), plan_s, exec_s,
                          fft_s, exec_s / fft_s);
            csv << line;
        }
    }
    return kOk;
}

// ---------------------------------------------------------------- cgstudy
int cmd_cgstudy(const Args& a) {
    const auto ns = values<std::size_t>(a, "n", {256, 1024}, [](const std::string& s) { return (std::size_t)to_u64(s, "--n"); });
    const auto gs = values<double>(a, "gamma", {0.0, 1.0 / 32, 1.0 / 8, 7.0 / 16}, [](const std::string& s) { return to_double(s, "--gamma"); });
    const double tol = a.has("tol") ? to_double(a.one("tol"), "--tol") : 2.2e-14;
    const double eps = a.has("eps") ? to_double(a.one("eps"), "--eps") : 2.2e-16;
    const unsigned trials = a.has("trials") ? (unsigned)to_u64(a.one("trials"), "--trials") : 5u;
    const std::uint64_t seed = a.has("seed") ? to_u64(a.one("seed"), "--seed") : 1u;
    auto csv = open_out(a.one("out"), "cgstudy");
    csv << "N,gamma,iterations,converged\n";
    nufft::GaussianSampler rng(seed);
    for (std::size_t n : ns)
        for (double g : gs) {
            if (!(g < 0.5)) {
                std::fprintf(stderr, "cgstudy: gamma must be < 1/2\n");
                return kDomain;
            }
            for (unsigned t = 0; t < trials; ++t) {
                std::vector<double> x;
                if (g == 0.0) {
                    x = nufft::worst_grid(n, 0.0);
                } else {  // equispaced + uniform perturbations of at most gamma (nufft_app.hpp:58-67)
                    x.resize(n);
                    for (std::size_t j = 0; j < n; ++j) {
                        const double d = g * (2.0 * rng.uniform() - 1.0);
                        x[j] = (static_cast<double>(j) + d) / static_cast<double>(n);
                    }
                    x[0] = g / static_cast<double>(n);
                    x = nufft::normalize_samples(x);
                }
                const nufft::Plan2 plan = nufft::plan_nufft2(x, eps);
                const nufft::ToeplitzOperator op = nufft::toeplitz_from_normal(plan);
                const auto f = rng.complex_vector(n);
                const nufft::CgReport rep = nufft::inufft2(plan, op, f, tol);
                char line[112];
                std::snprintf(line, sizeof line, "%zu,%.17g,%zu,%d\n", n, g, rep.iterations, rep.converged ? 1 : 0);
                csv << line;
            }
        }
    return kOk;
}

void usage() {
    std::fprintf(stderr,
                 "usage: nufft transform --type {1|2|3|2d2|inv1|inv2} --in FILE... --out FILE [--eps E] [--tol T]\n"
                 "                       [--threads N] [--seed S] [--fft]\n"
                 "       nufft verify  [--n N...] [--gamma G...] [--eps E...] [--trials T] [--seed S] [--decay] --out FILE\n"
                 "       nufft bench   [--n N...] [--eps E...] [--gamma G] [--trials T] [--seed S] --out FILE\n"
                 "       nufft cgstudy [--n N...] [--gamma G...] [--tol T] [--eps E] [--trials T] [--seed S] --out FILE\n");
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return kIo;
    }
    const std::string sub = argv[1];
    if (sub == "-h" || sub == "--help") {
        usage();
        return kOk;
    }
    try {
        if (sub == "transform")
            return cmd_transform(parse(argc, argv, 2, {"type", "in", "out", "eps", "tol", "threads", "seed"}, {"fft"}));
        if (sub == "verify")
            return cmd_verify(parse(argc, argv, 2, {"n", "gamma", "eps", "trials", "seed", "out"}, {"decay"}));
        if (sub == "bench")
            return cmd_bench(parse(argc, argv, 2, {"n", "eps", "gamma", "trials", "seed", "out"}, {}));
        if (sub == "cgstudy")
            return cmd_cgstudy(parse(argc, argv, 2, {"n", "gamma", "tol", "eps", "trials", "seed", "out"}, {}));
        throw Usage("unknown subcommand '" + sub + "'");
    } catch (const Usage& e) {
        std::fprintf(stderr, "nufft: %s\n", e.what());
        usage();
        return kIo;
    } catch (const nufft::CsvError& e) {
        std::fprintf(stderr, "nufft: %s\n", e.what());
        return kIo;
    } catch (const std::domain_error& e) {
        std::fprintf(stderr, "nufft: %s\n", e.what());
        return kDomain;
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "nufft: %s\n", e.what());
        return kDomain;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "nufft: %s\n", e.what());
        return kIo;
    }
}
