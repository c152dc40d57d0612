// oracle/synth_capi.cpp -- TEST / BENCH INFRASTRUCTURE, not product.
// The synthetic-corpus generator of the product tree (paper_2206_05269_b200/csrc/synth.cpp: plain host C++,
// recipe pinned in SURVEY.md 8(d)) compiled on its own into oracle/libwfsynth.so, so that the reference arm of
// bench.py (`--impl reference`) can build the SAME bytes without mapping the CUDA library into its process.
#include "../paper_2206_05269_b200/csrc/synth.cpp"

extern "C" {
__attribute__((visibility("default")))
int wfs_corpus_strided(uint64_t seed, uint64_t doc_begin, uint64_t doc_stride, uint64_t n_docs, uint32_t vocab,
                       double zipf_s, uint32_t speaker, uint64_t doc_bytes, uint8_t* out, int threads) {
    return wfcu::synth_corpus_strided(seed, doc_begin, doc_stride, n_docs, vocab, zipf_s, speaker, doc_bytes, out, threads);
}
__attribute__((visibility("default")))
int wfs_uniform(uint64_t seed, uint64_t n, int as_f64, void* out) { return wfcu::synth_uniform(seed, n, as_f64, out); }
}
