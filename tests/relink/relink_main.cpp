// tests/relink/relink_main.cpp -- TEST INFRASTRUCTURE for INTEGRATION.md section 1.
// A caller written against the reference's headers only -- the wordcount / compare flows of proj/src/cli.cpp:79-104,
// 176-230 without the CLI11 option parsing (that vendored header is not shipped) -- linked with the reference's OWN
// report.cpp (compiled unmodified from where it lies, against its own wfc/report.hpp) and, for everything else, with
// libwfc_b200.so: the relink a maintainer would do.  Prints what `wfc wordcount --format tsv|json` / `wfc compare`
// print.
#include <filesystem>
#include <iostream>
#include <string>
#include <vector>

#include "wfc/analysis.hpp"
#include "wfc/pipeline.hpp"
#include "wfc/report.hpp"

int main(int argc, char** argv) {
    using namespace wfc;
    if (argc < 4) {
        std::cerr << "usage: relink_demo wordcount <dir> <workers> [tsv|json] | compare <workers> <label=dir>...\n";
        return 2;
    }
    try {
        const std::string cmd = argv[1];
        if (cmd == "wordcount") {
            const std::string dir = argv[2];
            const std::size_t workers = std::stoul(argv[3]);
            const std::string format = argc > 4 ? argv[4] : "tsv";
            const std::string label = std::filesystem::path(dir).filename().string();
            Corpus corpus = ingest_directory(dir, label);
            RunResult run = run_wordcount(corpus.documents, workers);
            FrequencyTable table = top_k(remove_stopwords(std::move(run.counts), {}), label, 25);
            if (format == "json") std::cout << frequency_json(table).dump() << '\n';
            else write_frequency_tsv(std::cout, table);
            write_timings_tsv(std::cerr, run.timings);
            return 0;
        }
        if (cmd == "compare") {
            const std::size_t workers = std::stoul(argv[2]);
            std::vector<std::string> labels;
            std::vector<CountMap> counts;
            for (int i = 3; i < argc; ++i) {
                const std::string spec = argv[i];
                const auto eq = spec.find('=');
                labels.push_back(spec.substr(0, eq));
                counts.push_back(run_wordcount(ingest_directory(spec.substr(eq + 1), labels.back()).documents, workers).counts);
            }
            for (std::size_t i = 0; i < counts.size(); ++i) {
                CountMap pooled;
                for (std::size_t o = 0; o < counts.size(); ++o)
                    if (o != i)
                        for (const auto& [w, c] : counts[o]) pooled[w] += c;
                write_compare_tsv(std::cout, top_k(counts[i], labels[i], 5), distinctive_words(counts[i], pooled, labels[i], 5));
            }
            return 0;
        }
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
    return 2;
}
