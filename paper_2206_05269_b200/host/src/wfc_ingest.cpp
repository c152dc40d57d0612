// wfc_ingest.cpp -- the step in front of the path: files of a directory -> Corpus (interface:
// /root/reference/proj/include/wfc/analysis.hpp:15-29, 63-66; behaviour: proj/src/analysis.cpp:33-56, 134-152).
// File reading is host work; the byte work -- replacing invalid UTF-8 with U+FFFD -- is ONE device pass over all
// the files of the directory: they are read back to back into one buffer with a newline (valid on its own, so no
// sequence can straddle two files) between them, sanitised together, and cut apart again at the newlines that
// were inserted (utf8_sanitize never creates or removes a newline).
#include <algorithm>
#include <cstdio>
#include <fstream>

#include "wfc/wfc_b200.hpp"

namespace wfc {

namespace {
namespace fs = std::filesystem;

bool is_text_file_name(const fs::path& p) {
    std::string ext = p.extension().string();
    for (char& c : ext) c = (c >= 'A' && c <= 'Z') ? char(c + 32) : c;
    return ext == ".txt" || ext == ".text";
}

// appends the file's bytes to `into`
void slurp(const fs::path& path, std::string& into) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw IngestError("cannot read file: " + path.string());
    char block[1 << 16];
    for (;;) {
        const std::size_t got = std::fread(block, 1, sizeof(block), f);
        into.append(block, got);
        if (got < sizeof(block)) break;
    }
    const bool failed = std::ferror(f) != 0;
    std::fclose(f);
    if (failed) throw IngestError("read failed: " + path.string());
}
}  // namespace

Corpus ingest_directory(const fs::path& dir, std::string label) {
    std::error_code ec;
    if (!fs::is_directory(dir, ec)) throw IngestError("not a readable directory: " + dir.string());
    std::vector<fs::path> names;
    for (const fs::directory_entry& e : fs::directory_iterator(dir))
        if (e.is_regular_file() && is_text_file_name(e.path())) names.push_back(e.path().filename());
    std::sort(names.begin(), names.end());

    // one buffer, one device pass; newline counts of the raw files tell where each sanitised file ends
    std::string raw;
    std::vector<std::size_t> newlines_in(names.size(), 0);
    for (std::size_t i = 0; i < names.size(); ++i) {
        const std::size_t before = raw.size();
        slurp(dir / names[i], raw);
        newlines_in[i] = std::size_t(std::count(raw.begin() + std::ptrdiff_t(before), raw.end(), '\n'));
        raw += '\n';
    }
    const std::string clean = raw.empty() ? std::string() : utf8_sanitize(raw);

    Corpus corpus;
    corpus.label = std::move(label);
    corpus.documents.reserve(names.size());
    std::size_t at = 0;
    for (std::size_t i = 0; i < names.size(); ++i) {
        std::size_t end = at;
        for (std::size_t seen = 0;; ++end) {          // the (newlines_in[i] + 1)-th newline from `at` is the separator
            if (clean[end] == '\n' && seen++ == newlines_in[i]) break;
        }
        corpus.documents.push_back({names[i].string(), clean.substr(at, end - at)});
        at = end + 1;
    }
    return corpus;
}

std::unordered_set<Word> load_stopwords(const fs::path& file) {
    std::ifstream probe(file);
    if (!probe) throw IngestError("cannot read stop-word file: " + file.string());
    probe.close();
    // lines only separate words (a newline is whitespace): one tokenizer call for the whole file
    std::string text;
    slurp(file, text);
    std::unordered_set<Word> stopwords;
    for (Word& w : tokenize({"stopwords", std::move(text)}).words) stopwords.insert(std::move(w));
    return stopwords;
}

CountMap remove_stopwords(CountMap counts, const std::unordered_set<Word>& stopwords) {
    std::erase_if(counts, [&](const auto& kv) { return stopwords.count(kv.first) != 0; });
    return counts;
}

}  // namespace wfc
