// lk_cli.cpp -- `loopkit_b200`, the reference CLI's registration commands on
// the B200 path (proj/tools/loopkit_main.cpp). Host C++ over the C ABI
// through the header-only shim (include/loopkit_b200/registration.hpp).
//
//   loopkit_b200 register --source a.ply --target b.ply [options]
//       cmd_register (loopkit_main.cpp:54-66, flags :276-291): prints the 4x4
//       with %.17g, then inlier_ratio and fitness; "no-alignment" + exit 2.
//   loopkit_b200 icp --source a.ply --target b.ply --init "16 numbers" [options]
//       point-to-plane refinement; prints the refined 4x4,
//       iterations, converged, correspondences, rmse and fitness.
//   loopkit_b200 register-icp --source a.ply --target b.ply [register + icp options]
//       global registration followed by ICP on the full clouds (config D).
//   loopkit_b200 evaluate --mode registration --est e.log --truth t.log [--frags DIR] [--rmse-max M]
//       cmd_evaluate_registration (loopkit_main.cpp:225-234): Table-I recall /
//       precision of a registration log (metrics.cpp:112-156). Host-only.
//
// Errors print "error: <what>" and exit 1 (loopkit_main.cpp:405-408). PLY
// input follows read_ply (proj/src/io.cpp:33-56, 66-190, 245-272): ascii or
// binary_little_endian, scalar vertex properties, x/y/z required, normals
// normalised (zero below 1e-12).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "loopkit_b200/registration.hpp"

namespace {

struct CliError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Vec3 {
    double x, y, z;
};
struct PointCloud {  // proj/include/loopkit/geometry.hpp:92-99
    std::vector<Vec3> positions;
    std::vector<Vec3> normals;
};
struct RegistrationParams {  // proj/include/loopkit/registration.hpp:17-32
    double leaf = 0.05;
    double normal_radius = 0.1;
    double feature_radius = 0.25;
    std::int64_t hypothesis_count = 4'000'000;
    double similarity_tau = 0.9;
    double d_max = 0.075;
    double min_inlier_ratio = 0.25;
    std::optional<double> max_fitness;
    double normal_angle_max = 30.0 * M_PI / 180.0;
    std::uint64_t seed = 0;
    int threads = 0;
};

// ---- PLY (proj/src/io.cpp) ---------------------------------------------------
bool next_line(const std::string& text, std::size_t& pos, std::string& line) {  // io.cpp:33-41
    if (pos >= text.size()) return false;
    std::size_t end = text.find('\n', pos);
    if (end == std::string::npos) end = text.size();
    line = text.substr(pos, end - pos);
    if (!line.empty() && line.back() == '\r') line.pop_back();
    pos = end + 1;
    return true;
}

int scalar_size(const std::string& type) {  // io.cpp:49-56
    if (type == "char" || type == "uchar" || type == "int8" || type == "uint8") return 1;
    if (type == "short" || type == "ushort" || type == "int16" || type == "uint16") return 2;
    if (type == "int" || type == "uint" || type == "int32" || type == "uint32") return 4;
    if (type == "float" || type == "float32") return 4;
    if (type == "double" || type == "float64") return 8;
    return 0;
}

struct PlyProperty {
    std::string name;
    int byte_size = 0;
    bool is_double = false;
};

PointCloud read_ply(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw CliError("cannot open " + path);
    std::string text((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    auto fail = [&](std::size_t line_no, const std::string& what) {
        return CliError(path + ":" + std::to_string(line_no) + ": " + what);
    };
    // header (io.cpp:66-141)
    std::size_t pos = 0, line_no = 0, count = 0;
    std::string line;
    bool binary = false, in_vertex = false, have_vertex = false, have_format = false, done = false;
    std::vector<PlyProperty> props;
    if (!next_line(text, pos, line)) throw fail(line_no, "empty file");
    line_no += 1;
    if (line != "ply") throw fail(line_no, "missing ply magic");
    while (!done && next_line(text, pos, line)) {
        line_no += 1;
        std::istringstream ss(line);
        std::string word;
        ss >> word;
        if (word.empty() || word == "comment" || word == "obj_info") continue;
        if (word == "format") {
            std::string fmt, version;
            ss >> fmt >> version;
            if (fmt == "ascii") binary = false;
            else if (fmt == "binary_little_endian") binary = true;
            else throw CliError(path + ": unsupported format " + fmt);
            have_format = true;
        } else if (word == "element") {
            std::string name;
            std::size_t c = 0;
            ss >> name >> c;
            if (!ss) throw fail(line_no, "malformed element line");
            if (name == "vertex") {
                in_vertex = have_vertex = true;
                count = c;
            } else {
                if (!have_vertex && c > 0) throw CliError(path + ": element '" + name + "' precedes vertex data");
                in_vertex = false;
            }
        } else if (word == "property") {
            if (!in_vertex) continue;
            std::string type;
            ss >> type;
            if (type == "list") throw CliError(path + ": list property on vertex element");
            PlyProperty p;
            p.byte_size = scalar_size(type);
            if (p.byte_size == 0) throw fail(line_no, "unknown property type " + type);
            p.is_double = p.byte_size == 8 && (type == "double" || type == "float64");
            ss >> p.name;
            if (!ss) throw fail(line_no, "malformed property line");
            props.push_back(p);
        } else if (word == "end_header") {
            if (!have_format) throw fail(line_no, "missing format line");
            if (!have_vertex) throw fail(line_no, "missing vertex element");
            done = true;
        } else {
            throw fail(line_no, "unknown header keyword " + word);
        }
    }
    if (!done) throw fail(line_no, "missing end_header");
    // vertex table (io.cpp:144-190)
    std::map<std::string, std::vector<double>> cols;
    for (const PlyProperty& p : props) cols[p.name].reserve(count);
    if (binary) {
        std::size_t record = 0;
        for (const PlyProperty& p : props) record += static_cast<std::size_t>(p.byte_size);
        if (pos + record * count > text.size()) throw fail(line_no, "binary payload truncated");
        const char* base = text.data() + pos;
        for (std::size_t i = 0; i < count; ++i) {
            const char* rec = base + i * record;
            for (const PlyProperty& p : props) {
                double value = 0.0;
                if (p.byte_size == 4 && !p.is_double) {
                    float v;
                    std::memcpy(&v, rec, 4);
                    value = static_cast<double>(v);
                } else if (p.is_double) {
                    std::memcpy(&value, rec, 8);
                } else {
                    std::int64_t v = 0;
                    std::memcpy(&v, rec, static_cast<std::size_t>(p.byte_size));
                    value = static_cast<double>(v);
                }
                cols[p.name].push_back(value);
                rec += p.byte_size;
            }
        }
    } else {
        for (std::size_t i = 0; i < count; ++i) {
            if (!next_line(text, pos, line)) throw fail(line_no, "vertex data truncated");
            line_no += 1;
            std::istringstream ss(line);
            for (const PlyProperty& p : props) {
                double value;
                if (!(ss >> value)) throw fail(line_no, "malformed vertex line");
                cols[p.name].push_back(value);
            }
        }
    }
    auto col = [&](const char* n) -> const std::vector<double>* {
        auto it = cols.find(n);
        return it == cols.end() ? nullptr : &it->second;
    };
    const auto *x = col("x"), *y = col("y"), *z = col("z");
    if (!x || !y || !z) throw fail(line_no, "vertex element lacks x/y/z");
    PointCloud cloud;
    cloud.positions.resize(count);
    for (std::size_t i = 0; i < count; ++i) cloud.positions[i] = {(*x)[i], (*y)[i], (*z)[i]};
    const auto *nx = col("nx"), *ny = col("ny"), *nz = col("nz");
    if (nx && ny && nz) {  // io.cpp:259-268
        cloud.normals.resize(count);
        for (std::size_t i = 0; i < count; ++i) {
            const Vec3 n{(*nx)[i], (*ny)[i], (*nz)[i]};
            const double len = std::sqrt((n.x * n.x + n.y * n.y) + n.z * n.z);
            cloud.normals[i] = len > 1e-12 ? Vec3{n.x / len, n.y / len, n.z / len} : Vec3{0.0, 0.0, 0.0};
        }
    }
    return cloud;
}

// ---- registration log + Table-I scoring (proj/src/io.cpp, metrics.cpp) ------
struct LogEntry {  // proj/include/loopkit/io.hpp:41-46
    int i = 0, j = 0, n = 0;
    double T[16] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};  // row-major 4x4
};

std::vector<LogEntry> read_registration_log(const std::string& path) {  // io.cpp:341-369
    std::ifstream f(path, std::ios::binary);
    if (!f) throw CliError("cannot open " + path);
    std::string text((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    auto fail = [&](std::size_t line_no, const std::string& what) {
        return CliError(path + ":" + std::to_string(line_no) + ": " + what);
    };
    std::vector<LogEntry> out;
    std::size_t pos = 0, line_no = 0;
    std::string line;
    while (next_line(text, pos, line)) {
        line_no += 1;
        const std::size_t first = line.find_first_not_of(" \t");
        if (first == std::string::npos || line[first] == '#') continue;
        LogEntry e;
        {
            std::istringstream ss(line);
            if (!(ss >> e.i >> e.j >> e.n)) throw fail(line_no, "expected header line 'i j n'");
        }
        for (int r = 0; r < 4; ++r) {
            if (!next_line(text, pos, line)) throw fail(line_no, "truncated matrix block");
            line_no += 1;
            std::istringstream ss(line);
            if (!(ss >> e.T[4 * r] >> e.T[4 * r + 1] >> e.T[4 * r + 2] >> e.T[4 * r + 3]))
                throw fail(line_no, "expected 4 matrix values");
        }
        out.push_back(e);
    }
    return out;
}

struct RegistrationScore {  // proj/include/loopkit/metrics.hpp:39-45
    double recall = 0.0, precision = 0.0;
    int correct = 0, truth_count = 0, result_count = 0;
};

// eval_registration (metrics.cpp:112-156): a result is correct when its
// (i, j) pair is in the truth log and the RMSE between the two transforms on
// the probe points (fragment j's cloud, else the 8 corners of a unit cube)
// is below rmse_max; each truth entry is credited at most once.
RegistrationScore eval_registration(const std::vector<LogEntry>& results, const std::vector<LogEntry>& truth,
                                    const std::vector<PointCloud>& probes, double rmse_max) {
    RegistrationScore score;
    score.truth_count = static_cast<int>(truth.size());
    score.result_count = static_cast<int>(results.size());
    if (truth.empty() || results.empty()) return score;
    static const Vec3 cube[8] = {{-0.5, -0.5, -0.5}, {0.5, -0.5, -0.5}, {-0.5, 0.5, -0.5}, {0.5, 0.5, -0.5},
                                 {-0.5, -0.5, 0.5},  {0.5, -0.5, 0.5},  {-0.5, 0.5, 0.5},  {0.5, 0.5, 0.5}};
    auto apply = [](const double* T, const Vec3& p) {  // RigidTransform::operator*, geometry.hpp:26
        return Vec3{((T[0] * p.x + T[1] * p.y) + T[2] * p.z) + T[3], ((T[4] * p.x + T[5] * p.y) + T[6] * p.z) + T[7],
                    ((T[8] * p.x + T[9] * p.y) + T[10] * p.z) + T[11]};
    };
    auto pair_rmse = [&](const LogEntry& est, const LogEntry& gt) {
        const Vec3* pts = cube;
        std::size_t count = 8;
        if (est.j >= 0 && static_cast<std::size_t>(est.j) < probes.size() &&
            !probes[static_cast<std::size_t>(est.j)].positions.empty()) {
            pts = probes[static_cast<std::size_t>(est.j)].positions.data();
            count = probes[static_cast<std::size_t>(est.j)].positions.size();
        }
        double sq = 0.0;
        for (std::size_t k = 0; k < count; ++k) {
            const Vec3 a = apply(est.T, pts[k]), b = apply(gt.T, pts[k]);
            const double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
            sq += (dx * dx + dy * dy) + dz * dz;
        }
        return std::sqrt(sq / static_cast<double>(count));
    };
    std::vector<char> credited(truth.size(), 0);
    for (const LogEntry& est : results) {
        for (std::size_t t = 0; t < truth.size(); ++t) {
            if (credited[t] || truth[t].i != est.i || truth[t].j != est.j) continue;
            if (pair_rmse(est, truth[t]) < rmse_max) {
                credited[t] = 1;
                score.correct += 1;
            }
            break;
        }
    }
    score.recall = static_cast<double>(score.correct) / static_cast<double>(truth.size());
    score.precision = static_cast<double>(score.correct) / static_cast<double>(results.size());
    return score;
}

std::vector<PointCloud> load_fragment_clouds(const std::string& dir) {  // loopkit_main.cpp:31-42
    std::vector<PointCloud> clouds;
    for (int i = 0;; ++i) {
        char name[32];
        std::snprintf(name, sizeof(name), "fragment_%04d.ply", i);
        const std::string p = dir + "/" + name;
        if (!std::ifstream(p).good()) break;
        clouds.push_back(read_ply(p));
    }
    if (clouds.empty()) throw CliError("no fragment_%04d.ply files in " + dir);
    return clouds;
}

// ---- arguments ---------------------------------------------------------------
struct Args {
    std::map<std::string, std::string> opt;
    bool has(const std::string& k) const { return opt.count(k) != 0; }
    std::string str(const std::string& k) const {
        auto it = opt.find(k);
        if (it == opt.end()) throw CliError("--" + k + " is required");
        return it->second;
    }
    double num(const std::string& k, double dflt) const {
        if (!has(k)) return dflt;
        char* end = nullptr;
        const double v = std::strtod(opt.at(k).c_str(), &end);
        if (!end || *end) throw CliError("--" + k + ": not a number: " + opt.at(k));
        return v;
    }
    std::int64_t integer(const std::string& k, std::int64_t dflt) const {
        if (!has(k)) return dflt;
        char* end = nullptr;
        const long long v = std::strtoll(opt.at(k).c_str(), &end, 10);
        if (!end || *end) throw CliError("--" + k + ": not an integer: " + opt.at(k));
        return v;
    }
};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& known) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0) throw CliError("unexpected argument " + k);
        k = k.substr(2);
        bool ok = false;
        for (const std::string& n : known) ok = ok || n == k;
        if (!ok) throw CliError("unknown option --" + k);
        if (i + 1 >= argc) throw CliError("--" + k + " needs a value");
        a.opt[k] = argv[++i];
    }
    return a;
}

const std::vector<std::string> kRegisterOpts = {"source", "target", "hypotheses", "seed", "leaf", "dmax",
                                                "normal-radius", "feature-radius", "similarity-tau",
                                                "min-inlier-ratio", "max-fitness", "normal-angle-max", "threads",
                                                "device"};
const std::vector<std::string> kIcpOpts = {"source", "target", "init", "max-dist", "iterations", "eps", "device"};

RegistrationParams reg_params(const Args& a) {  // loopkit_main.cpp:280-291
    RegistrationParams p;
    p.hypothesis_count = a.integer("hypotheses", p.hypothesis_count);
    p.seed = static_cast<std::uint64_t>(a.integer("seed", static_cast<std::int64_t>(p.seed)));
    p.leaf = a.num("leaf", p.leaf);
    p.d_max = a.num("dmax", p.d_max);
    p.normal_radius = a.num("normal-radius", p.normal_radius);
    p.feature_radius = a.num("feature-radius", p.feature_radius);
    p.similarity_tau = a.num("similarity-tau", p.similarity_tau);
    p.min_inlier_ratio = a.num("min-inlier-ratio", p.min_inlier_ratio);
    const double mf = a.num("max-fitness", -1.0);
    if (mf >= 0.0) p.max_fitness = mf;
    p.normal_angle_max = a.num("normal-angle-max", p.normal_angle_max);
    p.threads = static_cast<int>(a.integer("threads", p.threads));
    return p;
}

void print_matrix(const double* R, const double* t) {  // loopkit_main.cpp:25-29
    for (int r = 0; r < 3; ++r)
        std::printf("%.17g %.17g %.17g %.17g\n", R[3 * r], R[3 * r + 1], R[3 * r + 2], t[r]);
    std::printf("%.17g %.17g %.17g %.17g\n", 0.0, 0.0, 0.0, 1.0);
}

int run_icp(const PointCloud& src, const PointCloud& tgt, const double* T0, const Args& a) {
    lk_cloud s = loopkit_b200::as_lk_cloud(src), t = loopkit_b200::as_lk_cloud(tgt);
    lk_icp_params p{};
    p.max_correspondence_distance = a.num("max-dist", 0.05);
    p.max_iterations = static_cast<int32_t>(a.integer("iterations", 30));
    p.convergence_eps = a.num("eps", 1e-10);
    p.device = static_cast<int32_t>(a.integer("device", -1));
    lk_icp_result r{};
    const lk_status st = lk_icp_point_to_plane(&s, &t, T0, &p, &r, nullptr);
    if (st != LK_OK) loopkit_b200::throw_status(st);
    print_matrix(r.R, r.t);
    std::printf("iterations %d\nconverged %d\ncorrespondences %lld\nrmse %.17g\nfitness %.17g\n", r.iterations,
                r.converged, static_cast<long long>(r.correspondences), r.rmse, r.fitness);
    return 0;
}

int usage() {
    std::fprintf(stderr,
                 "usage: loopkit_b200 register --source A.ply --target B.ply [--hypotheses N] [--seed S] [--leaf L]\n"
                 "                     [--dmax D] [--normal-radius R] [--feature-radius R] [--similarity-tau T]\n"
                 "                     [--min-inlier-ratio M] [--max-fitness F] [--normal-angle-max RAD]\n"
                 "                     [--threads N] [--device G]\n"
                 "       loopkit_b200 icp --source A.ply --target B.ply --init \"m00 m01 ... m33\" [--max-dist D]\n"
                 "                     [--iterations N] [--eps E] [--device G]\n"
                 "       loopkit_b200 register-icp --source A.ply --target B.ply [register options]\n"
                 "                     [--max-dist D] [--iterations N] [--eps E]\n"
                 "       loopkit_b200 evaluate --mode registration --est E.log --truth T.log [--frags DIR]\n"
                 "                     [--rmse-max M]\n");
    return 1;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    try {
        if (cmd == "register") {  // cmd_register, loopkit_main.cpp:54-66
            const Args a = parse(argc, argv, 2, kRegisterOpts);
            const PointCloud source = read_ply(a.str("source"));
            const PointCloud target = read_ply(a.str("target"));
            const RegistrationParams params = reg_params(a);
            auto result = loopkit_b200::register_global(source, target, params);
            if (!result) {
                std::printf("no-alignment\n");
                return 2;
            }
            print_matrix(result->transform.R, result->transform.t);
            std::printf("inlier_ratio %.17g\nfitness %.17g\n", result->inlier_ratio, result->fitness);
            return 0;
        }
        if (cmd == "icp") {
            const Args a = parse(argc, argv, 2, kIcpOpts);
            const PointCloud source = read_ply(a.str("source"));
            const PointCloud target = read_ply(a.str("target"));
            std::istringstream ss(a.str("init"));
            double m[16];
            for (double& v : m)
                if (!(ss >> v)) throw CliError("--init needs 16 numbers (row-major 4x4)");
            const double T0[12] = {m[0], m[1], m[2], m[4], m[5], m[6], m[8], m[9], m[10], m[3], m[7], m[11]};
            return run_icp(source, target, T0, a);
        }
        if (cmd == "register-icp") {
            std::vector<std::string> known = kRegisterOpts;
            for (const char* k : {"max-dist", "iterations", "eps"}) known.push_back(k);
            const Args a = parse(argc, argv, 2, known);
            const PointCloud source = read_ply(a.str("source"));
            const PointCloud target = read_ply(a.str("target"));
            auto result = loopkit_b200::register_global(source, target, reg_params(a));
            if (!result) {
                std::printf("no-alignment\n");
                return 2;
            }
            double T0[12];
            for (int k = 0; k < 9; ++k) T0[k] = result->transform.R[k];
            for (int k = 0; k < 3; ++k) T0[9 + k] = result->transform.t[k];
            return run_icp(source, target, T0, a);
        }
        if (cmd == "evaluate") {  // cmd_evaluate_registration, loopkit_main.cpp:225-234, flags :349-361
            const Args a = parse(argc, argv, 2, {"mode", "est", "truth", "frags", "rmse-max"});
            const std::string mode = a.str("mode");
            if (mode != "registration")
                throw CliError("--mode " + mode + ": only 'registration' is on the B200 path");
            std::vector<PointCloud> probes;
            if (a.has("frags") && !a.str("frags").empty()) probes = load_fragment_clouds(a.str("frags"));
            const RegistrationScore s = eval_registration(read_registration_log(a.str("est")),
                                                          read_registration_log(a.str("truth")), probes,
                                                          a.num("rmse-max", 0.2));
            std::printf("recall %.17g\nprecision %.17g\ncorrect %d\n", s.recall, s.precision, s.correct);
            return 0;
        }
        if (cmd == "-h" || cmd == "--help") {
            usage();
            return 0;
        }
        std::fprintf(stderr, "unknown command '%s'\n", cmd.c_str());
        return usage();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
