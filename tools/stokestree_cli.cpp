// stokestree -- command-line front end with the reference's flag set
// (proj/tools/stokestree_cli.cpp:33-65), parsed by hand (CLI11 is not in this image),
// running the B200 treecode through the drop-in harness (stokestree/bench.hpp).
// Exit codes as the reference: 1 invalid argument, 2 any other error.
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <string>

#include "stokestree/bench.hpp"

namespace st = stokestree;

static const char* kUsage =
    "stokestree - treecode summation of Stokeslet/stresslet velocities (B200)\n"
    "Modes: tree (treecode only), direct (reference sum only), both (adds the\n"
    "relative error E and the speedup of the treecode over the direct sum).\n"
    "  --testcase sphere|cube|file   particle source (default cube)\n"
    "  --n N            particle count (cube)        --levels L   sphere refinements, N = 20*4^L\n"
    "  --seed S         generator seed (default 0)   --density D  cube number density (2500)\n"
    "  --input PATH     particle file (file)         --order p    Taylor order (6)\n"
    "  --theta T        MAC parameter in (0,1) (0.5) --n0 N0      leaf capacity (2000)\n"
    "  --shrink auto|on|off (auto)                   --mode tree|direct|both (both)\n"
    "  --workers W      accepted, results identical  --devices G  GPUs (1)\n"
    "  --kernels stokeslet|stresslet|both|auto (auto)\n"
    "  --direct-sample S  time the direct sum on S evenly spaced targets (0 = all)\n"
    "  --out PATH  --format csv|human (human)  --dump-particles PATH\n";

int main(int argc, char** argv) {
    std::map<std::string, std::string> opt = {{"testcase", "cube"}, {"mode", "both"}, {"shrink", "auto"},
                                              {"kernels", "auto"}, {"format", "human"}};
    const std::map<std::string, bool> known = {
        {"testcase", 1}, {"n", 1}, {"levels", 1}, {"seed", 1}, {"density", 1}, {"input", 1},
        {"order", 1}, {"theta", 1}, {"n0", 1}, {"shrink", 1}, {"mode", 1}, {"workers", 1},
        {"kernels", 1}, {"direct-sample", 1}, {"out", 1}, {"format", 1}, {"dump-particles", 1}, {"devices", 1}};
    try {
        for (int i = 1; i < argc; ++i) {
            std::string a = argv[i];
            if (a == "--help" || a == "-h") {
                std::cout << kUsage;
                return 0;
            }
            if (a.rfind("--", 0) != 0) throw std::invalid_argument("unexpected argument '" + a + "'");
            a = a.substr(2);
            std::string v;
            const auto eq = a.find('=');
            if (eq != std::string::npos) {
                v = a.substr(eq + 1);
                a = a.substr(0, eq);
            } else {
                if (i + 1 >= argc) throw std::invalid_argument("--" + a + " needs a value");
                v = argv[++i];
            }
            if (!known.count(a)) throw std::invalid_argument("unknown option --" + a);
            opt[a] = v;
        }
        auto member = [&](const std::string& k, std::initializer_list<const char*> allowed) {
            for (const char* x : allowed)
                if (opt[k] == x) return;
            throw std::invalid_argument("--" + k + ": '" + opt[k] + "' not allowed");
        };
        member("testcase", {"sphere", "cube", "file"});
        member("mode", {"tree", "direct", "both"});
        member("shrink", {"auto", "on", "off"});
        member("kernels", {"stokeslet", "stresslet", "both", "auto"});
        member("format", {"csv", "human"});
        auto num = [&](const std::string& k, auto def) -> decltype(def) {
            if (!opt.count(k)) return def;
            try {
                std::size_t used = 0;
                if constexpr (std::is_floating_point_v<decltype(def)>) {
                    const double v = std::stod(opt[k], &used);
                    if (used != opt[k].size()) throw std::invalid_argument("");
                    return v;
                } else {
                    const long long v = std::stoll(opt[k], &used);
                    if (used != opt[k].size()) throw std::invalid_argument("");
                    return static_cast<decltype(def)>(v);
                }
            } catch (const std::exception&) {
                throw std::invalid_argument("--" + k + ": not a number: '" + opt[k] + "'");
            }
        };
        st::RunConfig cfg;
        cfg.params.order = num("order", cfg.params.order);
        cfg.params.theta = num("theta", cfg.params.theta);
        cfg.params.leaf_capacity = num("n0", cfg.params.leaf_capacity);
        cfg.params.workers = num("workers", cfg.params.workers);
        cfg.params.devices = num("devices", cfg.params.devices);
        cfg.cube.density = num("density", cfg.cube.density);
        cfg.direct_sample = num("direct-sample", (long long)0);
        const uint64_t seed = num("seed", (long long)0);
        const std::string tc = opt["testcase"];
        if (tc == "sphere") {
            cfg.testcase = st::TestCase::sphere;
            const int levels = num("levels", -1);
            if (levels < 0) throw std::invalid_argument("sphere test case needs --levels");
            cfg.sphere.levels = levels;
            cfg.sphere.seed = seed;
        } else if (tc == "cube") {
            cfg.testcase = st::TestCase::cube;
            const long long n = num("n", (long long)-1);
            if (n < 1) throw std::invalid_argument("cube test case needs --n");
            cfg.cube.n = static_cast<std::size_t>(n);
            cfg.cube.seed = seed;
        } else {
            cfg.testcase = st::TestCase::file;
            cfg.input_path = opt.count("input") ? opt["input"] : "";
        }
        cfg.mode = opt["mode"] == "tree" ? st::RunMode::tree
                 : opt["mode"] == "direct" ? st::RunMode::direct
                                           : st::RunMode::both;
        if (opt["shrink"] != "auto") cfg.shrink_override = opt["shrink"] == "on";
        if (opt["kernels"] == "stokeslet") cfg.kernels_override = st::KernelSelection::stokeslet_only();
        if (opt["kernels"] == "stresslet") cfg.kernels_override = st::KernelSelection::stresslet_only();
        if (opt["kernels"] == "both") cfg.kernels_override = st::KernelSelection::both();
        cfg.format = opt["format"] == "csv" ? st::ReportFormat::csv : st::ReportFormat::human;
        if (opt.count("out")) cfg.output_path = opt["out"];
        if (opt.count("dump-particles")) cfg.dump_particles_path = opt["dump-particles"];

        const st::RunResult res = st::run(cfg);
        std::ofstream file_out;
        std::ostream* out = &std::cout;
        if (!cfg.output_path.empty()) {
            file_out.open(cfg.output_path);
            if (!file_out) throw std::runtime_error("cannot open " + cfg.output_path.string());
            out = &file_out;
        }
        if (cfg.format == st::ReportFormat::csv) st::write_csv(*out, res.report);
        else st::write_human(*out, res);
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    }
    return 0;
}
