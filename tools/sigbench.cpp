// sigbench for the B200 path: the reference CLI's flags and output
// (/root/reference/proj/tools/sigbench.cpp:15-85), timing the GPU kernels via
// sigkit::run_grid (include/sigkit/bench.hpp). Built by
// paper_2501_08455_b200/build.py into tools/sigbench.
#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "sigkit/bench.hpp"
#include "sigkit/errors.hpp"

namespace {

template <typename T>
std::vector<T> parse_list(const std::string& s) {
    std::vector<T> out;
    std::stringstream ss(s);
    std::string item;
    while (std::getline(ss, item, ',')) {
        if (item.empty()) continue;
        std::stringstream is(item);
        T v{};
        if (!(is >> v)) throw sigkit::DomainError("bad list entry: " + item);
        out.push_back(v);
    }
    return out;
}

int usage() {
    std::cerr << "usage: sigbench [--batch-sizes a,b] [--seq-lens a,b] [--dims a,b] [--depths a,b]\n"
                 "                [--kernels sequential,parallel] [--repeats R] [--warmup W] [--dtype f64|f32]\n"
                 "                [--format csv|markdown] [--out FILE] [--seed S] [--paper-grid]\n";
    return 2;
}

}  // namespace

int main(int argc, char** argv) {
    sigkit::BenchConfig config;
    std::vector<std::string> kernel_names{"sequential", "parallel"};
    std::string dtype = "f64", format = "csv", out_path;
    bool paper_grid = false;
    try {
        for (int i = 1; i < argc; ++i) {
            const std::string a = argv[i];
            auto next = [&]() -> std::string {
                if (i + 1 >= argc) throw sigkit::DomainError("missing value for " + a);
                return argv[++i];
            };
            if (a == "--batch-sizes") config.batch_sizes = parse_list<std::size_t>(next());
            else if (a == "--seq-lens") config.seq_lens = parse_list<std::size_t>(next());
            else if (a == "--dims") config.dims = parse_list<int>(next());
            else if (a == "--depths") config.depths = parse_list<int>(next());
            else if (a == "--kernels") kernel_names = parse_list<std::string>(next());
            else if (a == "--repeats") config.repeats = std::atoi(next().c_str());
            else if (a == "--warmup") config.warmup = std::atoi(next().c_str());
            else if (a == "--dtype") dtype = next();
            else if (a == "--format") format = next();
            else if (a == "--out") out_path = next();
            else if (a == "--seed") config.seed = std::strtoull(next().c_str(), nullptr, 10);
            else if (a == "--paper-grid") paper_grid = true;
            else if (a == "--help" || a == "-h") return usage();
            else throw sigkit::DomainError("unknown option " + a);
        }
        if (config.repeats < 1 || config.warmup < 0) throw sigkit::DomainError("--repeats >= 1, --warmup >= 0");
        if (dtype != "f64" && dtype != "f32") throw sigkit::DomainError("--dtype must be f64 or f32");
        if (format != "csv" && format != "markdown") throw sigkit::DomainError("--format must be csv or markdown");
        for (std::size_t v : config.batch_sizes)
            if (v == 0) throw sigkit::DomainError("--batch-sizes entries must be positive");
        for (std::size_t v : config.seq_lens)
            if (v == 0) throw sigkit::DomainError("--seq-lens entries must be positive");
        for (int v : config.dims)
            if (v < 1) throw sigkit::DomainError("--dims entries must be positive");
        for (int v : config.depths)
            if (v < 1) throw sigkit::DomainError("--depths entries must be positive");
        config.kernels.clear();
        for (const std::string& k : kernel_names) config.kernels.push_back(sigkit::kernel_from_name(k));
        config.dtype = dtype == "f32" ? sigkit::Dtype::F32 : sigkit::Dtype::F64;
        if (paper_grid) config.points = sigkit::paper_grid_points(config.dims.front());
        const auto records = sigkit::run_grid(config);
        const auto fmt = format == "markdown" ? sigkit::BenchFormat::Markdown : sigkit::BenchFormat::Csv;
        if (out_path.empty()) sigkit::emit(records, fmt, std::cout);
        else sigkit::emit(records, fmt, out_path);
        std::size_t skipped = 0;
        for (const auto& r : records) skipped += r.skipped ? 1 : 0;
        if (skipped > 0)
            std::cerr << skipped << " of " << records.size() << " rows skipped on capacity grounds (empty stats)\n";
        std::cerr << "(B200: every kernel name runs the sm_100a path; times are CUDA-event kernel times)\n";
    } catch (const std::exception& err) {
        std::cerr << "error: " << err.what() << '\n';
        return 1;
    }
    return 0;
}
