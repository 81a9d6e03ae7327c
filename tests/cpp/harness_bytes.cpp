// Byte-level behaviour of the harness layer (write_csv, read_csv, write_human): compiled
// once against the reference's bench.hpp and once against this repo's drop-in headers;
// tests/test_cli_harness.py requires identical output.  Host-only: no GPU call is made.
#include <iostream>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "stokestree/bench.hpp"

using namespace stokestree;

static void try_read(const std::string& text) {
    std::istringstream in(text);
    try {
        const BenchReport r = read_csv(in);
        std::cout << "read ok: " << r.rows.size() << " rows\n";
        write_csv(std::cout, r);
    } catch (const std::runtime_error& e) {
        std::cout << "runtime_error: " << e.what() << '\n';
    } catch (const std::exception& e) {
        std::cout << "other exception: " << e.what() << '\n';
    }
}

int main() {
    BenchReport rep;
    BenchRow a;
    a.n = 1000000;
    a.p = 8;
    a.theta = 0.5;
    a.n0 = 2000;
    a.workers = 16;
    a.time_direct_s = 9707.0123456789;
    a.time_tree_s = 0.0606;
    a.speedup = 160000.5;
    a.error = 2.83e-5;
    a.farfield_evals = 143295410;
    a.direct_evals = 25699586242ull;
    rep.rows.push_back(a);
    BenchRow b;  // tree-only row: every optional empty
    b.n = 7;
    b.p = 0;
    b.theta = 0.1;
    b.n0 = 1;
    b.workers = 1;
    rep.rows.push_back(b);
    BenchRow c = a;
    c.theta = 1.0 / 3.0;
    c.time_direct_s.reset();
    c.error = 1e-300;
    c.speedup = std::numeric_limits<double>::infinity();
    c.time_tree_s = -0.0;
    rep.rows.push_back(c);

    std::cout << "== write_csv\n";
    write_csv(std::cout, rep);
    std::cout << "== round trip\n";
    std::stringstream ss;
    write_csv(ss, rep);
    const BenchReport back = read_csv(ss);
    std::cout << (back == rep ? "equal" : "different") << '\n';

    std::cout << "== read_csv errors\n";
    try_read("");
    try_read("N,p\n");
    try_read(std::string(kCsvHeader) + "\n");
    try_read(std::string(kCsvHeader) + "\n\n5,1,0.5,10,1,,,,,3,4\n\n");
    try_read(std::string(kCsvHeader) + "\n5,1,0.5,10,1,,,,3,4\n");
    try_read(std::string(kCsvHeader) + "\n5,1,0.5,10,1,,,,,3,4,9\n");
    try_read(std::string(kCsvHeader) + "\n5,1,0.5,10,1,,,,,3,4\n6,x,0.5,10,1,,,,,3,4\n");
    try_read(std::string(kCsvHeader) + "\n5,1,0.5,10,1,1e400,,,,3,4\n");
    try_read(std::string(kCsvHeader) + "\n5,1,0.5,10,1,,,,,3,\n");
    try_read(std::string(kCsvHeader) + "\r\n");

    std::cout << "== write_human\n";
    RunResult res;
    res.report = rep;
    res.selection = KernelSelection::both();
    res.n = 1000000;
    res.direct_targets = {0, 1000, 2000};
    VelocityResult vr;
    vr.time_build_s = 0.00105;
    vr.time_moments_s = 0.0015;
    vr.time_traverse_s = 0.0585;
    vr.time_total_s = 0.0606;
    res.tree = vr;
    write_human(std::cout, res);
    res.selection = KernelSelection::stokeslet_only();
    res.direct_targets.resize(1000000);
    write_human(std::cout, res);
    RunResult only_tree;
    BenchRow t = b;
    t.time_tree_s = 0.25;
    only_tree.report.rows.push_back(t);
    only_tree.selection = KernelSelection::stresslet_only();
    only_tree.tree = vr;
    write_human(std::cout, only_tree);
    RunResult only_direct;
    BenchRow d = b;
    d.time_direct_s = 12.5;
    only_direct.report.rows.push_back(d);
    only_direct.n = 7;
    only_direct.direct_targets = {0, 1, 2, 3, 4, 5, 6};
    write_human(std::cout, only_direct);
    return 0;
}
