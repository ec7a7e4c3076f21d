// capi.cpp -- the extern "C" boundary declared in include/graphlet_b200.h.
// Exceptions never cross it: each entry point maps the gl:: exception classes
// (mirrors of the reference's) to GL_ERR_* codes and a thread-local message.
#include "graphlet_b200.h"

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "graph.cuh"

namespace gl {
std::vector<u64> parse_edge_list(const char* text, size_t len);
std::vector<u64> parse_edge_list_file(const std::string& path);
std::vector<u64> generate_rmat_host(const RmatParams& p, u64 count);
std::vector<u64> generate_gnm(u64 n, u64 m, u64 seed);
std::vector<u64> generate_ba(u64 n, u32 k, u64 seed);
} // namespace gl

struct gl_graph {
    gl::Graph* g = nullptr;
};

namespace {

thread_local std::string t_err;
thread_local uint64_t t_line = 0;

template <typename F> int guarded(F&& f) {
    try {
        t_err.clear();
        t_line = 0;
        f();
        return GL_OK;
    } catch (const gl::parse_error& e) {
        t_err = e.what();
        t_line = e.line;
        return GL_ERR_PARSE;
    } catch (const gl::invalid_argument& e) {
        t_err = e.what();
        return GL_ERR_INVALID;
    } catch (const gl::io_error& e) {
        t_err = e.what();
        return GL_ERR_IO;
    } catch (const gl::oom_error& e) {
        t_err = e.what();
        return GL_ERR_OOM;
    } catch (const gl::cuda_error& e) {
        t_err = e.what();
        return GL_ERR_CUDA;
    } catch (const gl::consistency_error& e) {
        t_err = e.what();
        return GL_ERR_CONSISTENCY;
    } catch (const gl::overflow_error& e) {
        t_err = e.what();
        return GL_ERR_OVERFLOW;
    } catch (const gl::state_error& e) {
        t_err = e.what();
        return GL_ERR_STATE;
    } catch (const std::bad_alloc& e) {
        t_err = "host allocation failed";
        return GL_ERR_OOM;
    } catch (const std::exception& e) {
        t_err = e.what();
        return GL_ERR_INVALID;
    }
}

void require_device(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        throw gl::cuda_error(std::string("no CUDA device available: ") +
                             (e == cudaSuccess ? "device count is 0" : cudaGetErrorString(e)));
    }
    if (device < 0 || device >= n) throw gl::invalid_argument("device ordinal out of range");
}

void export_pairs(std::vector<gl::u64>&& v, uint64_t** pairs, uint64_t* count) {
    if (!pairs || !count) throw gl::invalid_argument("null output pointer");
    *count = v.size() / 2;
    *pairs = static_cast<uint64_t*>(std::malloc((v.size() ? v.size() : 1) * sizeof(uint64_t)));
    if (!*pairs) throw std::bad_alloc();
    if (!v.empty()) std::memcpy(*pairs, v.data(), v.size() * sizeof(uint64_t));
}

gl::Graph& G(const gl_graph* g) {
    if (!g || !g->g) throw gl::invalid_argument("null graph");
    return *g->g;
}

void to_c(const gl::u128* src, gl_u128* dst, int k) {
    for (int i = 0; i < k; ++i) {
        dst[i].lo = (uint64_t)src[i];
        dst[i].hi = (uint64_t)(src[i] >> 64);
    }
}

template <typename T> void d2h(T* host, const T* dev, size_t count, cudaStream_t s) {
    if (!count) return;
    GL_CUDA(cudaMemcpyAsync(host, dev, count * sizeof(T), cudaMemcpyDeviceToHost, s));
    GL_CUDA(cudaStreamSynchronize(s));
}

} // namespace

extern "C" {

const char* gl_last_error(void) { return t_err.c_str(); }
uint64_t gl_last_error_line(void) { return t_line; }
const char* gl_version(void) { return "graphlet_b200 0.1 (sm_100a)"; }
void gl_free(void* p) { std::free(p); }

int gl_set_overlap(int on) {
    gl::g_overlap.store(on ? 1 : 0);
    return GL_OK;
}

int gl_trim_device_cache(void) {
    return guarded([&] { gl::pool_trim(); });
}

int gl_load_edge_list(const char* text, size_t len, uint64_t** pairs, uint64_t* count) {
    return guarded([&] {
        if (!text && len) throw gl::invalid_argument("null text");
        export_pairs(gl::parse_edge_list(text, len), pairs, count);
    });
}

int gl_load_edge_list_file(const char* path, uint64_t** pairs, uint64_t* count) {
    return guarded([&] {
        if (!path) throw gl::invalid_argument("null path");
        export_pairs(gl::parse_edge_list_file(path), pairs, count);
    });
}

int gl_parse_edge_list_device(const char* text, size_t len, int device, uint64_t** pairs, uint64_t* count) {
    return guarded([&] {
        if (!text && len) throw gl::invalid_argument("null text");
        require_device(device);
        gl::DevBuf d;
        const gl::u64 k = gl::parse_edge_list_device(text, len, device, d, nullptr);
        std::vector<gl::u64> host(2 * k);
        if (k) GL_CUDA(cudaMemcpy(host.data(), d.p, 2 * k * sizeof(gl::u64), cudaMemcpyDeviceToHost));
        export_pairs(std::move(host), pairs, count);
    });
}

int gl_graph_build_text(const char* text, size_t len, int device, gl_graph** out) {
    return guarded([&] {
        if (!out) throw gl::invalid_argument("null output pointer");
        if (!text && len) throw gl::invalid_argument("null text");
        require_device(device);
        gl::DevBuf d;
        const gl::u64 k = gl::parse_edge_list_device(text, len, device, d, nullptr);
        if (!k) d.alloc(16);
        auto* h = new gl_graph;
        try {
            h->g = gl::build_graph_device(d.as<gl::u64>(), k, device);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int gl_generate_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c, uint64_t seed,
                     uint64_t** pairs, uint64_t* count) {
    return guarded([&] {
        gl::RmatParams p = gl::make_rmat_params(scale, a, b, c, seed);
        export_pairs(gl::generate_rmat_host(p, (gl::u64)edge_factor << scale), pairs, count);
    });
}

int gl_generate_rmat_device(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                            uint64_t seed, int device, uint64_t* d_pairs, uint64_t count) {
    return guarded([&] {
        require_device(device);
        gl::RmatParams p = gl::make_rmat_params(scale, a, b, c, seed);
        if (count != ((gl::u64)edge_factor << scale)) throw gl::invalid_argument("count != edge_factor << scale");
        GL_CUDA(cudaSetDevice(device));
        gl::generate_rmat_device(p, count, d_pairs, nullptr);
        GL_CUDA(cudaDeviceSynchronize());
    });
}

int gl_generate_gnm(uint64_t n, uint64_t m, uint64_t seed, uint64_t** pairs, uint64_t* count) {
    return guarded([&] { export_pairs(gl::generate_gnm(n, m, seed), pairs, count); });
}

int gl_generate_ba(uint64_t n, uint32_t attach, uint64_t seed, uint64_t** pairs, uint64_t* count) {
    return guarded([&] { export_pairs(gl::generate_ba(n, attach, seed), pairs, count); });
}

int gl_graph_build(const uint64_t* pairs, uint64_t count, int device, gl_graph** out) {
    return guarded([&] {
        if (!out) throw gl::invalid_argument("null output");
        if (!pairs && count) throw gl::invalid_argument("null pairs");
        require_device(device);
        GL_CUDA(cudaSetDevice(device));
        gl::DevBuf d;
        d.alloc((2 * count + 1) * sizeof(uint64_t));
        if (count) GL_CUDA(cudaMemcpy(d.p, pairs, 2 * count * sizeof(uint64_t), cudaMemcpyHostToDevice));
        auto* h = new gl_graph;
        try {
            h->g = gl::build_graph_device(d.as<gl::u64>(), count, device);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int gl_graph_build_device(const uint64_t* d_pairs, uint64_t count, int device, gl_graph** out) {
    return guarded([&] {
        if (!out) throw gl::invalid_argument("null output");
        if (!d_pairs && count) throw gl::invalid_argument("null pairs");
        require_device(device);
        auto* h = new gl_graph;
        try {
            h->g = gl::build_graph_device(d_pairs, count, device);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

void gl_graph_free(gl_graph* g) {
    if (!g) return;
    if (g->g) {
        cudaSetDevice(g->g->device);
        delete g->g;
    }
    delete g;
}

uint64_t gl_graph_num_vertices(const gl_graph* g) { return g && g->g ? g->g->d.n : 0; }
uint64_t gl_graph_num_edges(const gl_graph* g) { return g && g->g ? g->g->d.m : 0; }
uint32_t gl_graph_max_degree(const gl_graph* g) { return g && g->g ? g->g->d.dmax : 0; }

int gl_graph_degrees(const gl_graph* g, uint32_t* degree) {
    return guarded([&] {
        auto& gr = G(g);
        GL_CUDA(cudaSetDevice(gr.device));
        d2h(degree, gr.d.deg, gr.d.n, gr.stream);
    });
}

int gl_graph_labels(const gl_graph* g, uint64_t* label) {
    return guarded([&] {
        auto& gr = G(g);
        GL_CUDA(cudaSetDevice(gr.device));
        d2h(label, gr.d.label, gr.d.n, gr.stream);
    });
}

int gl_graph_csr(const gl_graph* g, uint64_t* offsets, uint32_t* adjacency) {
    return guarded([&] {
        auto& gr = G(g);
        GL_CUDA(cudaSetDevice(gr.device));
        if (offsets) d2h(offsets, gr.d.off, gr.d.n + 1, gr.stream);
        if (adjacency) d2h(adjacency, gr.d.adj, 2 * gr.d.m, gr.stream);
    });
}

int gl_orient_edges(const gl_graph* g, uint32_t* v, uint32_t* u) {
    return guarded([&] {
        auto& gr = G(g);
        GL_CUDA(cudaSetDevice(gr.device));
        if (v) d2h(v, gr.d.ev, gr.d.m, gr.stream);
        if (u) d2h(u, gr.d.eu, gr.d.m, gr.stream);
    });
}

int gl_global_from_unrestricted(const gl_unrestricted* c, uint64_t n, uint64_t m, gl_graphlet_vector* X) {
    return guarded([&] {
        if (!c || !X) throw gl::invalid_argument("null argument");
        gl::u128 C[17], XX[18];
        for (int i = 0; i < 17; ++i) C[i] = ((gl::u128)c->c[i].hi << 64) | c->c[i].lo;
        gl::global_from_unrestricted(C, n, m, XX);
        to_c(XX, X->x, 18);
    });
}

uint64_t gl_partials_len(const gl_graph* g, int world) {
    if (!g || !g->g || world < 1) return 0;
    gl::u64 m = g->g->d.m;
    return ((m + world - 1) / world) * (gl::u64)world;
}

int gl_count_begin(gl_graph* g, int rank, int world, int64_t* d_partials, void* stream) {
    return guarded([&] {
        auto& gr = G(g);
        if (!d_partials && gr.d.m) throw gl::invalid_argument("null partials");
        gl::count_begin(gr, rank, world, reinterpret_cast<gl::i64*>(d_partials),
                        static_cast<cudaStream_t>(stream));
    });
}

int gl_count_mid(gl_graph* g, int64_t* d_partials, void* stream) {
    return guarded([&] {
        auto& gr = G(g);
        gl::count_mid(gr, reinterpret_cast<gl::i64*>(d_partials), static_cast<cudaStream_t>(stream));
    });
}

int gl_triangle_counts_device(gl_graph* g, uint32_t** d_t, uint64_t* count) {
    return guarded([&] {
        auto& gr = G(g);
        if (!gr.cs.began) throw gl::state_error("gl_triangle_counts_device before gl_count_begin");
        if (d_t) *d_t = gr.cs.t.as<uint32_t>();
        if (count) *count = gr.d.m;
    });
}

int gl_count_finish(gl_graph* g, const int64_t* d_partials, uint64_t edge_begin, uint64_t edge_end,
                    gl_unrestricted* unres, void* stream) {
    return guarded([&] {
        auto& gr = G(g);
        if (!unres) throw gl::invalid_argument("null unres");
        gl::u128 C[17];
        gl::count_finish(gr, reinterpret_cast<const gl::i64*>(d_partials), edge_begin, edge_end, C,
                         static_cast<cudaStream_t>(stream));
        to_c(C, unres->c, 17);
    });
}

int gl_count(gl_graph* g, gl_graphlet_vector* X, gl_unrestricted* unres) {
    return guarded([&] {
        auto& gr = G(g);
        if (!X) throw gl::invalid_argument("null X");
        GL_CUDA(cudaSetDevice(gr.device));
        const gl::u64 m = gr.d.m;
        gr.cs.part.alloc((2 * m + 2) * sizeof(gl::i64));
        gl::count_begin(gr, 0, 1, gr.cs.part.as<gl::i64>(), gr.stream);
        gl::count_mid(gr, gr.cs.part.as<gl::i64>(), gr.stream);
        gl::u128 C[17], XX[18];
        gl::count_finish(gr, gr.cs.part.as<gl::i64>(), 0, m, C, gr.stream);
        gl::global_from_unrestricted(C, gr.d.n, m, XX);
        to_c(XX, X->x, 18);
        if (unres) to_c(C, unres->c, 17);
    });
}

int gl_count_edges(gl_graph* g, gl_graphlet_vector* X, gl_unrestricted* unres, uint32_t* t, uint64_t* x7,
                   uint64_t* x10) {
    return guarded([&] {
        auto& gr = G(g);
        if (!X) throw gl::invalid_argument("null X");
        GL_CUDA(cudaSetDevice(gr.device));
        const gl::u64 m = gr.d.m;
        gr.cs.part.alloc((2 * m + 2) * sizeof(gl::i64));
        gr.cs.out_t = t;
        gr.cs.out_x7 = x7;
        struct Reset { // the early-copy pointers never outlive this call
            gl::CountState& cs;
            ~Reset() {
                if (cs.s3) cudaStreamSynchronize(cs.s3);
                cs.out_t = nullptr;
                cs.out_x7 = nullptr;
            }
        } reset{gr.cs};
        gl::count_begin(gr, 0, 1, gr.cs.part.as<gl::i64>(), gr.stream);
        gl::count_mid(gr, gr.cs.part.as<gl::i64>(), gr.stream);
        gl::u128 C[17], XX[18];
        gl::count_finish(gr, gr.cs.part.as<gl::i64>(), 0, m, C, gr.stream);
        if (x10 && m)
            GL_CUDA(cudaMemcpyAsync(x10, gr.cs.x10.p, m * sizeof(uint64_t), cudaMemcpyDeviceToHost, gr.stream));
        GL_CUDA(cudaStreamSynchronize(gr.stream));
        if (gr.cs.s3) GL_CUDA(cudaStreamSynchronize(gr.cs.s3));
        gl::global_from_unrestricted(C, gr.d.n, m, XX);
        to_c(XX, X->x, 18);
        if (unres) to_c(C, unres->c, 17);
    });
}

int gl_micro_records(const gl_graph* g, uint64_t first, uint64_t count, gl_micro_record* out) {
    return guarded([&] {
        auto& gr = G(g);
        if (!out && count) throw gl::invalid_argument("null output");
        static_assert(sizeof(gl_micro_record) == 10 * sizeof(uint64_t), "record layout");
        gl::micro_records(gr, first, count, reinterpret_cast<gl::u64*>(out));
    });
}

int gl_edge_motif_records(const gl_graph* g, uint64_t first, uint64_t count, gl_edge_motif_record* out) {
    return guarded([&] {
        auto& gr = G(g);
        if (!out && count) throw gl::invalid_argument("null output");
        static_assert(sizeof(gl_edge_motif_record) == 5 * sizeof(uint64_t), "record layout");
        gl::edge_motif_records(gr, first, count, reinterpret_cast<gl::u64*>(out));
    });
}

int gl_edge_counts(const gl_graph* g, uint64_t first, uint64_t count, uint32_t* t, uint64_t* x7,
                   uint64_t* x10) {
    return guarded([&] {
        auto& gr = G(g);
        const auto& cs = gr.cs;
        if (!cs.have_micro) throw gl::state_error("no counts computed yet");
        if (first < cs.shard_begin || first > cs.shard_end || count > cs.shard_end - first)
            throw gl::invalid_argument("edge range outside the computed shard");
        GL_CUDA(cudaSetDevice(gr.device));
        // the three copies queue back to back, one synchronisation
        if (count && t)
            GL_CUDA(cudaMemcpyAsync(t, cs.t.as<uint32_t>() + first, count * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                    gr.stream));
        if (count && x7)
            GL_CUDA(cudaMemcpyAsync(x7, cs.x7.as<uint64_t>() + first, count * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                    gr.stream));
        if (count && x10)
            GL_CUDA(cudaMemcpyAsync(x10, cs.x10.as<uint64_t>() + first, count * sizeof(uint64_t),
                                    cudaMemcpyDeviceToHost, gr.stream));
        GL_CUDA(cudaStreamSynchronize(gr.stream));
    });
}

int gl_edge_counts_device(const gl_graph* g, const uint32_t** t, const uint64_t** x7, const uint64_t** x10) {
    return guarded([&] {
        auto& gr = G(g);
        if (!gr.cs.have_micro) throw gl::state_error("no counts computed yet");
        if (t) *t = gr.cs.t.as<uint32_t>();
        if (x7) *x7 = gr.cs.x7.as<uint64_t>();
        if (x10) *x10 = gr.cs.x10.as<uint64_t>();
    });
}

int gl_last_timings(const gl_graph* g, float ms[5], uint32_t* launches) {
    return guarded([&] {
        auto& gr = G(g);
        for (int i = 0; i < 5; ++i) ms[i] = gr.cs.ms[i];
        if (launches) *launches = gr.cs.launches;
    });
}

int gl_last_work(const gl_graph* g, uint64_t work[4]) {
    return guarded([&] {
        auto& gr = G(g);
        for (int i = 0; i < 4; ++i) work[i] = gr.cs.work[i];
    });
}

int gl_cycle_pieces(const gl_graph* g, uint32_t* out, uint64_t cap, uint64_t* count_total) {
    return guarded([&] {
        auto& gr = G(g);
        if (!gr.cs.began) throw gl::state_error("no gl_count_begin yet");
        const uint64_t n = gr.cs.cycle_pieces;
        if (count_total) *count_total = n;
        const uint64_t k = n < cap ? n : cap;
        if (!out || !k) return;
        GL_CUDA(cudaSetDevice(gr.device));
        if (gr.cs.s2) GL_CUDA(cudaStreamSynchronize(gr.cs.s2));
        GL_CUDA(cudaStreamSynchronize(gr.stream));
        GL_CUDA(cudaMemcpy(out, gr.cs.pieces.p, k * 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    });
}

} // extern "C"
