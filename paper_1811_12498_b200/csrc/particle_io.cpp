// Particle text format (particle_io.hpp:30-126), host side: header line naming the
// present blocks ("x", optionally "f" and/or "h nu"), then one row per particle with
// three fields per block written with 17 significant digits ("%.17g"), so a write /
// read round trip is bit-exact.  Errors carry the reference's messages and line numbers.
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "stokestree_c.h"

namespace st {
st_status io_set_error(st_status s, const std::string& m);  // capi.cu
}

namespace {

struct IoError {
    st_status s;
    std::string m;
};

bool finite3(const double* a) { return std::isfinite(a[0]) && std::isfinite(a[1]) && std::isfinite(a[2]); }

// validate(ps, sel) (particles.hpp:41-70), host side (the writer runs on the host)
void validate_host(const st_particles* ps, bool sto, bool str) {
    if (!sto && !str) throw IoError{ST_INVALID_ARGUMENT, "kernel selection: at least one kernel must be enabled"};
    if (!ps || ps->n == 0) throw IoError{ST_INVALID_ARGUMENT, "particle set is empty"};
    auto check = [&](const double* a, const char* name) {
        if (!a) throw IoError{ST_INVALID_ARGUMENT, std::string("particle array '") + name + "' has mismatched length"};
        for (size_t i = 0; i < ps->n; ++i)
            if (!finite3(a + 3 * i))
                throw IoError{ST_INVALID_ARGUMENT, std::string("particle array '") + name + "' contains a non-finite value"};
    };
    check(ps->position, "position");
    if (sto) check(ps->force_weight, "force_weight");
    if (str) {
        check(ps->dipole_weight, "dipole_weight");
        check(ps->normal, "normal");
        for (size_t i = 0; i < ps->n; ++i) {
            const double* v = ps->normal + 3 * i;
            const double len = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
            if (std::abs(len - 1.0) > 1e-12)
                throw IoError{ST_INVALID_ARGUMENT, "normal " + std::to_string(i) + " is not unit length"};
        }
    }
}

}  // namespace

struct st_loaded {
    size_t n = 0;
    bool f = false, h = false;
    std::vector<double> pos, fw, hw, nu;
};

extern "C" st_status st_write_particles(const char* path, const st_particles* ps, int stokeslet, int stresslet) {
    try {
        const bool sto = stokeslet != 0, str = stresslet != 0;
        validate_host(ps, sto, str);
        std::FILE* fp = std::fopen(path, "w");
        if (!fp) throw IoError{ST_RUNTIME_ERROR, std::string("write_particles: cannot open ") + path};
        std::string header = "x";
        if (sto) header += " f";
        if (str) header += " h nu";
        std::fprintf(fp, "%s\n", header.c_str());
        char buf[32];
        auto put = [&](const double* v, bool first) {
            for (int c = 0; c < 3; ++c) {
                std::snprintf(buf, sizeof buf, "%.17g", v[c]);
                if (!(first && c == 0)) std::fputc(' ', fp);
                std::fputs(buf, fp);
            }
        };
        for (size_t i = 0; i < ps->n; ++i) {
            put(ps->position + 3 * i, true);
            if (sto) put(ps->force_weight + 3 * i, false);
            if (str) {
                put(ps->dipole_weight + 3 * i, false);
                put(ps->normal + 3 * i, false);
            }
            std::fputc('\n', fp);
        }
        const bool bad = std::ferror(fp) != 0;
        std::fclose(fp);
        if (bad) throw IoError{ST_RUNTIME_ERROR, std::string("write_particles: write failed for ") + path};
        return st::io_set_error(ST_OK, "");
    } catch (const IoError& e) {
        return st::io_set_error(e.s, e.m);
    }
}

extern "C" st_status st_read_particles(const char* path, st_loaded** out, size_t* n, int* stokeslet,
                                       int* stresslet) {
    try {
        if (!out) throw IoError{ST_INVALID_ARGUMENT, "read_particles: null output"};
        *out = nullptr;
        std::ifstream in(path);
        if (!in) throw IoError{ST_RUNTIME_ERROR, std::string("read_particles: cannot open ") + path};
        std::string header;
        if (!std::getline(in, header))
            throw IoError{ST_RUNTIME_ERROR, std::string("read_particles: missing header line in ") + path};
        std::istringstream hs(header);
        std::vector<std::string> blocks;
        for (std::string tok; hs >> tok;) blocks.push_back(tok);
        bool has_f = false, has_h = false, has_nu = false;
        if (blocks.empty() || blocks[0] != "x")
            throw IoError{ST_RUNTIME_ERROR, "read_particles: header must start with 'x' (line 1)"};
        for (size_t i = 1; i < blocks.size(); ++i) {
            if (blocks[i] == "f" && !has_f) has_f = true;
            else if (blocks[i] == "h" && !has_h) has_h = true;
            else if (blocks[i] == "nu" && !has_nu) has_nu = true;
            else throw IoError{ST_RUNTIME_ERROR, "read_particles: bad header block '" + blocks[i] + "' (line 1)"};
        }
        if (has_h != has_nu)
            throw IoError{ST_RUNTIME_ERROR, "read_particles: blocks 'h' and 'nu' must appear together (line 1)"};
        if (!has_f && !has_h)
            throw IoError{ST_RUNTIME_ERROR, "read_particles: header declares no weight blocks (line 1)"};
        auto* L = new st_loaded();
        L->f = has_f;
        L->h = has_h;
        const int fields = 3 * (1 + (has_f ? 1 : 0) + (has_h ? 2 : 0));
        std::string line;
        size_t lineno = 1;
        try {
            while (std::getline(in, line)) {
                ++lineno;
                if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
                std::istringstream ls(line);
                double v[12];
                for (int c = 0; c < fields; ++c)
                    if (!(ls >> v[c]))
                        throw IoError{ST_RUNTIME_ERROR, "read_particles: expected " + std::to_string(fields) +
                                                            " fields (line " + std::to_string(lineno) + ")"};
                std::string extra;
                if (ls >> extra)
                    throw IoError{ST_RUNTIME_ERROR,
                                  "read_particles: trailing fields (line " + std::to_string(lineno) + ")"};
                int c = 0;
                L->pos.insert(L->pos.end(), v + c, v + c + 3);
                c += 3;
                if (has_f) {
                    L->fw.insert(L->fw.end(), v + c, v + c + 3);
                    c += 3;
                }
                if (has_h) {
                    L->hw.insert(L->hw.end(), v + c, v + c + 3);
                    L->nu.insert(L->nu.end(), v + c + 3, v + c + 6);
                }
            }
            L->n = L->pos.size() / 3;
            if (L->n == 0) throw IoError{ST_RUNTIME_ERROR, std::string("read_particles: no particle rows in ") + path};
        } catch (...) {
            delete L;
            throw;
        }
        *out = L;
        if (n) *n = L->n;
        if (stokeslet) *stokeslet = has_f;
        if (stresslet) *stresslet = has_h;
        return st::io_set_error(ST_OK, "");
    } catch (const IoError& e) {
        return st::io_set_error(e.s, e.m);
    }
}

extern "C" st_status st_loaded_copy(const st_loaded* L, double* pos, double* f, double* h, double* nu) {
    if (!L) return st::io_set_error(ST_INVALID_ARGUMENT, "loaded particles: null");
    auto cp = [](const std::vector<double>& src, double* dst) {
        if (dst && !src.empty()) std::memcpy(dst, src.data(), src.size() * sizeof(double));
    };
    cp(L->pos, pos);
    cp(L->fw, f);
    cp(L->hw, h);
    cp(L->nu, nu);
    return ST_OK;
}

extern "C" void st_loaded_free(st_loaded* L) { delete L; }
