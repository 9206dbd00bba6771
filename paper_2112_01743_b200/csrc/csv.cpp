// CSV writers of the drop-in (include/chebpr/csv.hpp; reference: src/csv.cpp:37-84).
// Output bytes are the reference's: same headers, "%.17g" data, "%.3f" timings, '\n'
// line ends; a file that cannot be opened or closed raises ParseError with the
// reference's texts ("cannot write <path>", "write failed for <path>").
//
// Rank files of n rows are formatted in parallel blocks (each block's text is built in
// memory, then written in order), so a 33 M-vertex rank file is not bound by one
// thread's printf.
#include "chebpr/csv.hpp"

#include <algorithm>
#include <cstring>
#include <thread>

#include "chebpr/errors.hpp"

namespace chebpr {

std::string fmt17(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

namespace {

// Owns an output file; close() reports a failed flush like the reference.
class OutFile {
public:
    explicit OutFile(const std::string& path) : path_(path), f_(std::fopen(path.c_str(), "wb")) {
        if (!f_) throw ParseError("cannot write " + path_);
    }
    ~OutFile() {
        if (f_) std::fclose(f_);
    }
    OutFile(const OutFile&) = delete;
    OutFile& operator=(const OutFile&) = delete;
    std::FILE* get() const { return f_; }
    void put(const std::string& s) { std::fwrite(s.data(), 1, s.size(), f_); }
    void close() {
        std::FILE* f = f_;
        f_ = nullptr;
        if (std::fclose(f) != 0) throw ParseError("write failed for " + path_);
    }

private:
    std::string path_;
    std::FILE* f_;
};

void append_row(std::string& s, long long id, double v) {
    char buf[64];
    const int k = std::snprintf(buf, sizeof buf, "%lld,%.17g\n", id, v);
    s.append(buf, (size_t)k);
}

}  // namespace

void write_ranks_csv(const std::string& path, const Vector& ranks) {
    OutFile out(path);
    out.put("vertex_id,rank\n");
    const int64_t n = ranks.size();
    constexpr int64_t kBlock = int64_t(1) << 18;  // rows per formatting block
    const int64_t blocks = (n + kBlock - 1) / kBlock;
    const int T = (int)std::max<int64_t>(1, std::min<int64_t>(blocks, std::max(1u, std::thread::hardware_concurrency())));
    for (int64_t b0 = 0; b0 < blocks; b0 += T) {  // T blocks at a time, written in order
        const int64_t nb = std::min<int64_t>(T, blocks - b0);
        std::vector<std::string> text((size_t)nb);
        auto fill = [&](int64_t j) {
            const int64_t lo = (b0 + j) * kBlock, hi = std::min(n, lo + kBlock);
            std::string& s = text[(size_t)j];
            s.reserve((size_t)(hi - lo) * 32);
            for (int64_t i = lo; i < hi; ++i) append_row(s, (long long)i, ranks[i]);
        };
        if (nb == 1) {
            fill(0);
        } else {
            std::vector<std::thread> th;
            for (int64_t j = 0; j < nb; ++j) th.emplace_back(fill, j);
            for (auto& t : th) t.join();
        }
        for (auto& s : text) out.put(s);
    }
    out.close();
}

void write_cpaa_trace_csv(const std::string& path, const std::vector<TraceRow>& trace, bool with_err) {
    OutFile out(path);
    out.put(std::string("k,c_k,S_k,residual_mass,elapsed_ms") + (with_err ? ",err\n" : "\n"));
    for (const TraceRow& r : trace) {
        std::string row = std::to_string(r.k) + "," + fmt17(r.c_k) + "," + fmt17(r.S_k) + "," +
                          fmt17(r.residual_mass) + ",";
        char ms[48];
        std::snprintf(ms, sizeof ms, "%.3f", r.elapsed_ms);
        row += ms;
        if (with_err) row += "," + fmt17(r.err);
        out.put(row + "\n");
    }
    out.close();
}

void write_power_trace_csv(const std::string& path, const std::vector<TraceRow>& trace, bool with_err) {
    OutFile out(path);
    out.put(std::string("k,l1_change,elapsed_ms") + (with_err ? ",err\n" : "\n"));
    for (const TraceRow& r : trace) {
        char ms[48];
        std::snprintf(ms, sizeof ms, "%.3f", r.elapsed_ms);
        std::string row = std::to_string(r.k) + "," + fmt17(r.l1_change) + "," + ms;
        if (with_err) row += "," + fmt17(r.err);
        out.put(row + "\n");
    }
    out.close();
}

void write_compare_csv(std::FILE* out, const std::vector<CompareRow>& rows) {
    std::fputs("algo,parallelism,rounds,err,l1,elapsed_ms\n", out);
    for (const CompareRow& r : rows) {
        char ms[48];
        std::snprintf(ms, sizeof ms, "%.3f", r.elapsed_ms);
        const std::string row = r.algo + "," + std::to_string(r.parallelism) + "," + std::to_string(r.rounds) +
                                "," + fmt17(r.err) + "," + fmt17(r.l1) + "," + ms + "\n";
        std::fputs(row.c_str(), out);
    }
}

void write_compare_csv(const std::string& path, const std::vector<CompareRow>& rows) {
    OutFile out(path);
    write_compare_csv(out.get(), rows);
    out.close();
}

}  // namespace chebpr
