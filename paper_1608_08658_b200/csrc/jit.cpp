// sfdb200-jit: puts the B200 backend under the reference's UNMODIFIED
// operators (sfd::seismic::forward / adjoint / gradient, verify::*).
//
// The reference runs every operator as one call of a JIT-compiled C kernel:
// codegen::generate emits the loop nest plus the trampoline
// `int <Name>_call(void **argv)` (proj/src/codegen.cpp:579-629), and
// runtime::compile_and_load compiles it with
//     $STENCILFD_CC -shared -fPIC <preset flags> -o <hash>.so <hash>.c -lm
// (proj/src/runtime.cpp:177-250), dlopens it and resolves `<Name>_call`.
// The problem constants (extents, nt, dt, h, taps, sparse-set sizes) exist
// only as literals in that source.  This driver reads them back from the
// source and compiles, instead of the loop nest, a shim
//     static const sfdb200_desc D = {...};
//     int <Name>_call(void **argv) { return sfdb200_call(&D, argv); }
// so the argv the reference binds (seismic.cpp:363-368) goes to the GPU.
//
// Two ways in, neither touching the reference:
//  * gcc wrapper (the "b200" preset, include/sfdb200/stencilfd_preset.hpp):
//    preset flags `-wrapper <this> -L<lib> -Wl,--no-as-needed -lsfdb200
//    -Wl,-rpath,<lib>`; gcc runs each sub-command through this program, which
//    swaps the generated source for the shim in the `cc1` step and passes
//    `as` / `collect2` through unchanged.  Other presets in the same process
//    keep compiling the reference's own C.
//  * STENCILFD_CC=<this> (the reference's documented compiler hook): every
//    kernel compile of the process goes to the GPU; this program then adds
//    the include / link flags itself and runs `cc` ($SFDB200_HOST_CC).
// A source that is not a generated stencilfd kernel passes through
// untouched; a stencilfd kernel that is not an acoustic operator (or cannot
// be read back) fails the compile with the reason on stderr, which
// compile_and_load reports as CompileError (runtime.cpp:216-221).
//
// `sfdb200-jit --describe <file.c>` prints the descriptor read from a source
// as JSON (tests/test_jit.py).
//
// Device: `-DSFDB200_DEVICE=<n>` among the flags (part of the JIT cache key).
// Gradient kernels get SFDB200_F_GRAD_NO_ROW2: the generated kernel leaves the
// t = 2 term to seismic::gradient's host loop (seismic.cpp:468-490).

#include <sys/wait.h>
#include <unistd.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <optional>
#include <regex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sfdb200.h"

namespace {

struct Parsed {
    std::string name;
    sfdb200_desc d{};
};

std::string read_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot read " + path);
    std::ostringstream s;
    s << f.rdbuf();
    return s.str();
}

bool is_stencilfd_kernel(const std::string& src) {
    static const std::regex call(R"(\nint (\w+)_call\(void \*\*argv\)\n)");
    return std::regex_search(src, call) && src.find("#include <math.h>") == 0;
}

std::vector<long> dims_of(const std::string& brackets) {
    std::vector<long> out;
    static const std::regex d(R"(\[(\d+)\])");
    for (auto it = std::sregex_iterator(brackets.begin(), brackets.end(), d);
         it != std::sregex_iterator(); ++it)
        out.push_back(std::stol((*it)[1]));
    return out;
}

double literal(const std::string& s) {
    char* end = nullptr;
    const double v = std::strtod(s.c_str(), &end);
    if (end == s.c_str() || *end) throw std::runtime_error("bad numeric literal '" + s + "'");
    return v;
}

// Reads the operator's descriptor back from a generated source
// (codegen::generate's fixed layout: signature, array casts, the time loop,
// the solved update and the sparse loops, codegen.cpp:247-265,348-462).
Parsed parse(const std::string& src, int device) {
    auto need = [](bool ok, const std::string& what) {
        if (!ok) throw std::runtime_error("sfdb200-jit: cannot read " + what + " from the kernel");
    };
    Parsed p;
    std::smatch m;
    static const std::regex call(R"(\nint (\w+)_call\(void \*\*argv\)\n)");
    need(std::regex_search(src, m, call), "the entry point");
    p.name = m[1];

    // Signature: grids, then sparse triples, then block sizes.
    const std::regex sig("\nint " + p.name + R"(\(([^)]*)\)\n)");
    need(std::regex_search(src, m, sig), "the signature");
    std::vector<std::string> grids, sets;
    {
        const std::string params = m[1];
        static const std::regex param(R"((double|long) \*?(\w+))");
        for (auto it = std::sregex_iterator(params.begin(), params.end(), param);
             it != std::sregex_iterator(); ++it) {
            const std::string name = (*it)[2];
            static const std::regex sparse(R"((\w+)_(idx|w|data)_vec)");
            std::smatch sm;
            if (std::regex_match(name, sm, sparse)) {
                if (sm[2] == "idx") sets.push_back(sm[1]);
            } else if (name.size() > 4 && name.compare(name.size() - 4, 4, "_vec") == 0) {
                grids.push_back(name.substr(0, name.size() - 4));
            }
        }
    }
    sfdb200_desc& d = p.d;
    const std::vector<std::string> fwd{"u", "m", "damp"}, adj{"v", "m", "damp"},
        grd{"v", "u", "m", "damp", "grad"};
    if (grids == fwd && sets == std::vector<std::string>{"src", "rec"}) {
        d.kind = SFDB200_FORWARD;
    } else if (grids == adj && sets == std::vector<std::string>{"src", "rec"}) {
        d.kind = SFDB200_ADJOINT;
    } else if (grids == grd && sets == std::vector<std::string>{"rec"}) {
        d.kind = SFDB200_GRADIENT;
        d.flags = SFDB200_F_GRAD_NO_ROW2;
    } else {
        throw std::runtime_error("sfdb200-jit: '" + p.name +
                                 "' is not a seismic forward / adjoint / gradient kernel "
                                 "(build_*_ir, seismic.cpp:241-331)");
    }
    const std::string f = d.kind == SFDB200_FORWARD ? "u" : "v";  // the propagated field

    // Extents from the casts: m is [P0][P1]..., cast as (*m)[P1]...; the
    // field's cast (*u)[P0][P1]... drops the row dim.
    need(std::regex_search(src, m, std::regex(R"(double \(\*m\)((?:\[\d+\])+) = )")),
         "the model extents");
    const std::vector<long> mdims = dims_of(m[1]);
    need(std::regex_search(src, m, std::regex("double \\(\\*" + f + R"(\)((?:\[\d+\])+) = )")),
         "the field extents");
    const std::vector<long> fdims = dims_of(m[1]);
    d.ndim = static_cast<int>(fdims.size());
    need((d.ndim == 2 || d.ndim == 3) && mdims.size() + 1 == fdims.size() &&
             std::equal(mdims.begin(), mdims.end(), fdims.begin() + 1),
         "consistent extents");
    for (int k = 0; k < d.ndim; ++k) d.padded[k] = fdims[static_cast<size_t>(k)];

    // Sparse-set sizes from the trace casts (*<set>_data)[npoints].
    for (const std::string& s : sets) {
        need(std::regex_search(src, m, std::regex("double \\(\\*" + s + R"(_data\)\[(\d+)\] = )")),
             "the size of set " + s);
        const long n = std::stol(m[1]);
        (s == "src" ? d.nsrc : d.nrec) = n;
        need(std::regex_search(src, m, std::regex("long \\(\\*" + s + R"(_idx\)\[(\d+)\] = )")) &&
                 std::stol(m[1]) == d.ndim,
             "the index width of set " + s);
    }

    // The solved update writes the field at the time index: `u[iT % 3][...] =`
    // (rolling slots) or `u[iT][...] =` (saved history); first touch writes 0.0.
    need(std::regex_search(src, m, std::regex("\\b" + f + R"(\[(i\d+)( % 3)?\]((?:\[i\d+\])+) = -)")),
         "the update statement");
    const std::string T = m[1];
    const bool rolling = m[2].matched;
    d.save = d.kind == SFDB200_FORWARD && !rolling;
    need(rolling || d.kind == SFDB200_FORWARD, "rolling adjoint slots");
    // The time loop: forward `for (int iT = 2; iT < nt; iT++)`, backward
    // `for (int iT = nt - 1; iT >= 2; iT--)` (lowering.hpp:78-80).
    if (std::regex_search(src, m, std::regex("for \\(int " + T + " = 2; " + T + R"( < (\d+); )" + T +
                                             R"(\+\+\))"))) {
        need(d.kind == SFDB200_FORWARD, "a forward time loop only in Forward");
        d.nt = std::stol(m[1]);
    } else if (std::regex_search(src, m, std::regex("for \\(int " + T + R"( = (\d+); )" + T +
                                                    " >= 2; " + T + R"(--\))"))) {
        need(d.kind != SFDB200_FORWARD, "a backward time loop only in Adjoint / Gradient");
        d.nt = std::stol(m[1]) + 1;
    } else {
        need(false, "the time loop");
    }

    // Space order: the largest spatial stencil offset [iK +- k] (iK != iT).
    long R = 0;
    {
        static const std::regex off(R"(\[(i\d+) [-+] (\d+)\])");
        for (auto it = std::sregex_iterator(src.begin(), src.end(), off);
             it != std::sregex_iterator(); ++it)
            if ((*it)[1] != T) R = std::max(R, std::stol((*it)[2]));
    }
    need(R >= 1 && R <= 8, "the stencil radius");
    d.space_order = static_cast<int>(2 * R);

    // dt: the injection scale dt^2 (`<set>_w[p][0]*<dt^2>*<set>_data[...]`,
    // codegen.cpp:436-449), else the damping coefficient 1/(2 dt) of the
    // update's denominator `/(<1/(2dt)>*tempD + <1/dt^2>*tempM)`.
    if (std::regex_search(src, m, std::regex(R"(_w\[p\]\[0\]\*)" + std::string(R"(([0-9][0-9.]*(?:e[-+]?\d+)?))") + R"(\*\w+_data\[)"))) {
        d.dt = std::sqrt(literal(m[1]));
    } else {
        need(std::regex_search(src, m, std::regex(R"(double (temp\d+) = damp\[)")), "the damping term");
        const std::string td = m[1];
        need(std::regex_search(src, m, std::regex(R"(/\(([0-9][0-9.]*(?:e[-+]?\d+)?)\*)" + td + R"( \+ )")),
             "the damping coefficient");
        d.dt = 1.0 / (2.0 * literal(m[1]));
    }
    // h: the offset-1 tap w_1 / h^2 of the Laplacian on the first spatial
    // index, w_1 from fd_coefficients(2, so) (sfdb200_fd2, bit-exact with fd.cpp).
    {
        const std::string tidx = rolling ? "\\(" + T + " [-+] 1\\) % 3" : T + " - 1";
        need(std::regex_search(src, m, std::regex(R"(([0-9][0-9.]*(?:e[-+]?\d+)?)\*)" + f + "\\[" + tidx +
                                                  R"(\]\[i\d+ - 1\])")),
             "the Laplacian taps");
        double w[17];
        need(sfdb200_fd2(d.space_order, w) == 0, "the FD weights");
        d.h = std::sqrt(w[R + 1] / literal(m[1]));
    }
    need(d.dt > 0 && std::isfinite(d.dt) && d.h > 0 && std::isfinite(d.h), "dt and h");
    d.device = device;
    return p;
}

std::string shim(const Parsed& p, const std::string& origin) {
    const sfdb200_desc& d = p.d;
    char buf[2048];
    std::snprintf(buf, sizeof buf,
                  "/* sfdb200 shim generated by sfdb200-jit from the stencilfd kernel %s:\n"
                  " * its <Name>_call(argv) goes to the B200 backend (include/sfdb200.h). */\n"
                  "#include <stdio.h>\n"
                  "#include \"sfdb200.h\"\n"
                  "static const sfdb200_desc D = {%d, %d, {%ld, %ld, %ld}, %d, %ld, %.17g, %.17g,\n"
                  "                               %ld, %ld, %d, %d, %d};\n"
                  "int %s_call(void **argv)\n{\n"
                  "  int rc = sfdb200_call(&D, argv);\n"
                  "  if (rc) fprintf(stderr, \"sfdb200: %%s\\n\", sfdb200_last_error());\n"
                  "  return rc;\n}\n",
                  origin.c_str(), d.kind, d.ndim, d.padded[0], d.padded[1],
                  d.ndim == 3 ? d.padded[2] : 0L, d.space_order, d.nt, d.dt, d.h, d.nsrc, d.nrec,
                  d.save, d.device, d.flags, p.name.c_str());
    return buf;
}

std::string json(const Parsed& p) {
    const sfdb200_desc& d = p.d;
    char buf[1024];
    std::snprintf(buf, sizeof buf,
                  "{\"name\": \"%s\", \"kind\": %d, \"ndim\": %d, \"padded\": [%ld, %ld, %ld], "
                  "\"space_order\": %d, \"nt\": %ld, \"dt\": %.17g, \"h\": %.17g, \"nsrc\": %ld, "
                  "\"nrec\": %ld, \"save\": %d, \"device\": %d, \"flags\": %d}",
                  p.name.c_str(), d.kind, d.ndim, d.padded[0], d.padded[1], d.padded[2],
                  d.space_order, d.nt, d.dt, d.h, d.nsrc, d.nrec, d.save, d.device, d.flags);
    return buf;
}

std::string self_dir() {
    char buf[4096];
    const ssize_t n = readlink("/proc/self/exe", buf, sizeof buf - 1);
    if (n <= 0) throw std::runtime_error("sfdb200-jit: cannot locate itself");
    buf[n] = 0;
    std::string s(buf);
    return s.substr(0, s.rfind('/'));  // <pkg>/bin
}

int device_of(const std::vector<std::string>& args) {
    for (const std::string& a : args)
        if (a.rfind("-DSFDB200_DEVICE=", 0) == 0) return std::atoi(a.c_str() + 17);
    return 0;
}

// Index of the generated kernel source among the arguments, if any.
std::optional<size_t> kernel_arg(const std::vector<std::string>& args, size_t from) {
    for (size_t i = from; i < args.size(); ++i) {
        const std::string& a = args[i];
        if (a.size() < 3 || a.compare(a.size() - 2, 2, ".c") != 0 || a[0] == '-') continue;
        if (i > 0 && (args[i - 1] == "-dumpbase" || args[i - 1] == "-o")) continue;
        if (access(a.c_str(), R_OK) != 0) continue;
        if (is_stencilfd_kernel(read_file(a))) return i;
    }
    return std::nullopt;
}

int run(const std::vector<std::string>& args) {
    std::vector<char*> av;
    for (const std::string& a : args) av.push_back(const_cast<char*>(a.c_str()));
    av.push_back(nullptr);
    const pid_t pid = fork();
    if (pid < 0) return 127;
    if (pid == 0) {
        execvp(av[0], av.data());
        std::perror(av[0]);
        _exit(127);
    }
    int status = 0;
    if (waitpid(pid, &status, 0) < 0) return 127;
    return WIFEXITED(status) ? WEXITSTATUS(status) : 128;
}

// Writes the shim for args[k] next to it and points args[k] at it.
std::string translate(std::vector<std::string>& args, size_t k) {
    const Parsed p = parse(read_file(args[k]), device_of(args));
    const std::string out = args[k] + ".sfdb200." + std::to_string(getpid()) + ".c";
    std::ofstream f(out);
    f << shim(p, args[k]);
    if (!f) throw std::runtime_error("sfdb200-jit: cannot write " + out);
    args[k] = out;
    return out;
}

}  // namespace

int main(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    try {
        if (args.size() == 2 && args[0] == "--describe") {
            std::printf("%s\n", json(parse(read_file(args[1]), 0)).c_str());
            return 0;
        }
        if (args.empty()) {
            std::fprintf(stderr, "usage: sfdb200-jit --describe <kernel.c> | (gcc -wrapper) | "
                                 "(STENCILFD_CC) <cc arguments>\n");
            return 2;
        }
        const std::string dir = self_dir();
        const std::string include = dir + "/../../include";
        const std::string lib = dir + "/..";
        if (args[0][0] != '-') {
            // gcc -wrapper: args = <sub-command> <its arguments>.
            const std::string& prog = args[0];
            const std::string base = prog.substr(prog.rfind('/') + 1);
            if (base != "cc1") return run(args);
            const std::optional<size_t> k = kernel_arg(args, 1);
            if (!k) return run(args);
            const std::string tmp = translate(args, *k);
            args.insert(args.begin() + 1, "-I" + include);
            const int rc = run(args);
            std::remove(tmp.c_str());
            return rc;
        }
        // STENCILFD_CC: args = -shared -fPIC <flags> -o <so> <c> -lm
        const char* cc = std::getenv("SFDB200_HOST_CC");
        std::vector<std::string> cmd{cc && *cc ? cc : "cc"};
        const std::optional<size_t> k = kernel_arg(args, 0);
        std::string tmp;
        if (k) {
            tmp = translate(args, *k);
            cmd.push_back("-I" + include);
        }
        cmd.insert(cmd.end(), args.begin(), args.end());
        if (k) {
            for (const char* a : {"-Wl,--no-as-needed", "-lsfdb200"}) cmd.emplace_back(a);
            cmd.push_back("-L" + lib);
            cmd.push_back("-Wl,-rpath," + lib);
        }
        const int rc = run(cmd);
        if (!tmp.empty()) std::remove(tmp.c_str());
        return rc;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 1;
    }
}
