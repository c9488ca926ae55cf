// saba drop-in (B200 / sm_100a) — immutable CSR graph.
// API of the reference's saba/graph.hpp. Canonicalisation runs in
// libsaba_cuda's host graph builder (parallel radix sort); the first GPU call
// on a Graph uploads one device replica (packed {base, degree} + adjacency)
// that lives as long as the Graph and its copies.
#pragma once

#include <algorithm>
#include <istream>
#include <map>
#include <memory>
#include <mutex>
#include <ostream>
#include <span>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "saba/common.hpp"

namespace saba {

struct LoadOptions {
    char comment_char = '#';
};

class Graph {
public:
    [[nodiscard]] uint32_t vertex_count() const noexcept { return n_; }
    [[nodiscard]] uint64_t edge_count() const noexcept { return m_; }

    [[nodiscard]] uint32_t degree(uint32_t u) const {
        check_arg(u < n_, "degree: vertex out of range");
        return offsets_[u + 1] - offsets_[u];
    }
    [[nodiscard]] std::span<const uint32_t> neighbors(uint32_t u) const {
        check_arg(u < n_, "neighbors: vertex out of range");
        return {adjacency_.data() + offsets_[u], adjacency_.data() + offsets_[u + 1]};
    }
    [[nodiscard]] bool has_edge(uint32_t u, uint32_t v) const {
        const auto nb = neighbors(u);
        return std::binary_search(nb.begin(), nb.end(), v);
    }
    [[nodiscard]] uint32_t slot_of(uint32_t u, uint32_t v) const {
        const auto nb = neighbors(u);
        const auto it = std::lower_bound(nb.begin(), nb.end(), v);
        check_arg(it != nb.end() && *it == v, "slot_of: not an edge");
        return offsets_[u] + uint32_t(it - nb.begin());
    }
    [[nodiscard]] uint32_t edge_index(uint32_t u, uint32_t v) const {
        const auto nb = neighbors(u);
        const auto it = std::lower_bound(nb.begin(), nb.end(), v);
        check_arg(it != nb.end() && *it == v, "edge_index: not an edge");
        return slot_edge_[offsets_[u] + uint32_t(it - nb.begin())];
    }
    [[nodiscard]] const uint32_t* offsets_data() const noexcept { return offsets_.data(); }
    [[nodiscard]] const uint32_t* adjacency_data() const noexcept { return adjacency_.data(); }
    [[nodiscard]] const std::vector<uint32_t>& offsets() const noexcept { return offsets_; }
    [[nodiscard]] const std::vector<uint32_t>& adjacency() const noexcept { return adjacency_; }
    [[nodiscard]] uint32_t slot_edge(uint32_t s) const noexcept { return slot_edge_[s]; }
    [[nodiscard]] std::pair<uint32_t, uint32_t> edge(uint32_t e) const { return edges_[e]; }
    [[nodiscard]] uint64_t original_id(uint32_t u) const { return original_ids_[u]; }
    [[nodiscard]] uint32_t max_degree() const noexcept { return max_degree_; }

    /// Canonicalising constructor: loops dropped, duplicates / reversals
    /// merged, n = max(n_hint, largest id + 1). `device` >= 0 (an extension;
    /// default host, as the reference) runs the canonicalisation on that GPU
    /// (saba_cu_graph_from_edges): the same CSR, built by a device sort.
    static Graph from_edges(uint32_t n_hint, std::vector<std::pair<uint32_t, uint32_t>> pairs,
                            int device = -1) {
        std::vector<uint32_t> flat;
        flat.reserve(2 * pairs.size());
        for (const auto& [a, b] : pairs) {
            flat.push_back(a);
            flat.push_back(b);
        }
        saba_hgraph* h = nullptr;
        if (device >= 0)
            detail::raise_on(saba_cu_graph_from_edges(n_hint, flat.data(), pairs.size(), 0, device, &h),
                             "from_edges");
        else
            detail::raise_on(saba_hgraph_from_edges(n_hint, flat.data(), pairs.size(), &h), "from_edges");
        Graph g;
        g.adopt(h);
        return g;
    }

    /// Adopt a CSR that is already canonical (sorted, symmetric, loop-free).
    static Graph from_csr(std::vector<uint32_t> offsets, std::vector<uint32_t> adjacency) {
        check_arg(!offsets.empty(), "from_csr: empty offsets");
        saba_hgraph* h = nullptr;
        detail::raise_on(saba_hgraph_from_csr(uint32_t(offsets.size() - 1), offsets.data(),
                                              adjacency.data(), &h),
                         "from_csr");
        saba_hgraph_free(h);
        Graph g;
        g.offsets_ = std::move(offsets);
        g.adjacency_ = std::move(adjacency);
        g.finish();
        return g;
    }

    /// SNAP-style text edge list: two non-negative integer labels per line,
    /// comment lines skipped, labels numbered in order of first appearance,
    /// self-loops dropped before numbering.
    static Graph load_edge_list(std::istream& in, const LoadOptions& options = {}) {
        std::unordered_map<uint64_t, uint32_t> id_of;
        std::vector<uint64_t> labels;
        std::vector<std::pair<uint32_t, uint32_t>> pairs;
        std::string line;
        for (uint64_t line_no = 1; std::getline(in, line); ++line_no) {
            const std::string where = "parse error at line " + std::to_string(line_no);
            size_t p = line.find_first_not_of(" \t\r");
            if (p == std::string::npos || line[p] == options.comment_char) continue;
            uint64_t lab[2];
            for (int t = 0; t < 2; ++t) {
                check_data(p != std::string::npos, where + ": expected two vertex ids");
                const size_t q = line.find_first_of(" \t\r", p);
                const std::string tok = line.substr(p, q == std::string::npos ? std::string::npos : q - p);
                check_data(!tok.empty() && tok.find_first_not_of("0123456789") == std::string::npos,
                           where + ": non-integer token '" + tok + "'");
                try {
                    lab[t] = std::stoull(tok);
                } catch (const std::exception&) {
                    check_data(false, where + ": vertex id out of range");
                }
                p = q == std::string::npos ? q : line.find_first_not_of(" \t\r", q);
            }
            check_data(p == std::string::npos, where + ": trailing tokens");
            if (lab[0] == lab[1]) continue;
            uint32_t ids[2];
            for (int t = 0; t < 2; ++t) {
                const auto [it, fresh] = id_of.emplace(lab[t], uint32_t(labels.size()));
                if (fresh) labels.push_back(lab[t]);
                ids[t] = it->second;
            }
            pairs.emplace_back(ids[0], ids[1]);
        }
        check_data(!labels.empty() && !pairs.empty(), "empty graph");
        Graph g = from_edges(uint32_t(labels.size()), std::move(pairs));
        check_data(g.edge_count() >= 1, "empty graph (no edges after canonicalization)");
        g.original_ids_ = std::move(labels);
        return g;
    }

    /// Edge list whose re-load reproduces this graph's ids: vertices are
    /// introduced in internal-id order (each by an edge to an already
    /// introduced neighbour, or paired with its first neighbour), then the
    /// remaining edges follow in edge-id order.
    void write_edge_list(std::ostream& out) const {
        std::vector<char> seen(n_, 0), used(m_, 0);
        for (uint32_t k = 0; k < n_; ++k) {
            if (seen[k]) continue;
            const auto nb = neighbors(k);
            const auto it = std::find_if(nb.begin(), nb.end(), [&](uint32_t j) { return seen[j] != 0; });
            if (it != nb.end()) {
                out << original_ids_[*it] << ' ' << original_ids_[k] << '\n';
                used[edge_index(k, *it)] = 1;
            } else {
                check_data(!nb.empty(), "write_edge_list: isolated vertices are not expressible");
                out << original_ids_[k] << ' ' << original_ids_[nb.front()] << '\n';
                seen[nb.front()] = 1;
                used[edge_index(k, nb.front())] = 1;
            }
            seen[k] = 1;
        }
        for (uint32_t e = 0; e < m_; ++e)
            if (!used[e]) out << original_ids_[edges_[e].first] << ' ' << original_ids_[edges_[e].second] << '\n';
    }

    /// The device replica on `device` (created on first use; shared by copies).
    /// Thread-safe: the reference's Graph may be read from any number of
    /// threads at once (graph.hpp:24-27), so the lazy creation is locked, and
    /// libsaba_cuda serialises calls on one handle (saba_cu_graph::mu).
    /// Handles live as long as the graph, so a pointer returned to one
    /// thread stays valid while another asks for a different device.
    saba_cu_graph* device_handle(int device = 0) const { return device_group({device}); }

    /// One replica per entry of `devices` behind a single handle
    /// (saba_cu_graph_create_multi; repeats = logical shards on one GPU).
    saba_cu_graph* device_group(const std::vector<int>& devices) const {
        std::lock_guard<std::mutex> lock(replicas_->mu);
        auto& slot = replicas_->by_devices[devices];
        if (!slot) {
            saba_cu_graph* h = nullptr;
            detail::raise_on(saba_cu_graph_create_multi(offsets_.data(), adjacency_.data(), n_, adjacency_.size(),
                                                        devices.data(), int(devices.size()), &h),
                             "graph upload");
            slot = std::make_unique<DeviceReplica>(h);
        }
        return slot->handle;
    }

private:
    struct DeviceReplica {
        saba_cu_graph* handle;
        explicit DeviceReplica(saba_cu_graph* h) : handle(h) {}
        DeviceReplica(const DeviceReplica&) = delete;
        ~DeviceReplica() { saba_cu_graph_destroy(handle); }
    };
    struct Replicas {
        std::mutex mu;
        std::map<std::vector<int>, std::unique_ptr<DeviceReplica>> by_devices;
    };

    void adopt(saba_hgraph* h) {
        n_ = saba_hgraph_vertex_count(h);
        offsets_.resize(size_t(n_) + 1);
        adjacency_.resize(2 * saba_hgraph_edge_count(h));
        const int rc = saba_hgraph_csr(h, offsets_.data(), adjacency_.data());
        saba_hgraph_free(h);
        detail::raise_on(rc, "csr");
        finish();
    }

    // Derived arrays: edge ids in sorted (u<v) order, slot -> edge id, labels.
    void finish() {
        n_ = uint32_t(offsets_.size() - 1);
        m_ = adjacency_.size() / 2;
        slot_edge_.assign(adjacency_.size(), 0);
        edges_.clear();
        edges_.reserve(m_);
        max_degree_ = 0;
        for (uint32_t u = 0; u < n_; ++u) {
            max_degree_ = std::max(max_degree_, offsets_[u + 1] - offsets_[u]);
            for (uint32_t s = offsets_[u]; s < offsets_[u + 1]; ++s)
                if (adjacency_[s] > u) {
                    slot_edge_[s] = uint32_t(edges_.size());
                    edges_.emplace_back(u, adjacency_[s]);
                }
        }
        for (uint32_t u = 0; u < n_; ++u)
            for (uint32_t s = offsets_[u]; s < offsets_[u + 1]; ++s)
                if (adjacency_[s] < u) slot_edge_[s] = slot_edge_[slot_of(adjacency_[s], u)];
        original_ids_.resize(n_);
        for (uint32_t u = 0; u < n_; ++u) original_ids_[u] = u;
    }

    uint32_t n_ = 0;
    uint64_t m_ = 0;
    uint32_t max_degree_ = 0;
    std::vector<uint32_t> offsets_, adjacency_, slot_edge_;
    std::vector<std::pair<uint32_t, uint32_t>> edges_;
    std::vector<uint64_t> original_ids_;
    std::shared_ptr<Replicas> replicas_ = std::make_shared<Replicas>();
};

/// Whether a BFS from vertex 0 reaches every vertex.
inline bool is_connected(const Graph& g) {
    const uint32_t n = g.vertex_count();
    if (n == 0) return false;
    std::vector<uint32_t> order{0};
    std::vector<char> hit(n, 0);
    hit[0] = 1;
    for (size_t i = 0; i < order.size(); ++i)
        for (uint32_t v : g.neighbors(order[i]))
            if (!hit[v]) {
                hit[v] = 1;
                order.push_back(v);
            }
    return order.size() == n;
}

/// 2-colouring per component with each component's first vertex on side 0;
/// {false, {}} as soon as an odd cycle is found.
inline std::pair<bool, std::vector<char>> bipartition(const Graph& g) {
    const uint32_t n = g.vertex_count();
    std::vector<char> side(n, -1);
    std::vector<uint32_t> order;
    for (uint32_t r = 0; r < n; ++r) {
        if (side[r] != -1) continue;
        side[r] = 0;
        order.assign(1, r);
        for (size_t i = 0; i < order.size(); ++i) {
            const uint32_t u = order[i];
            for (uint32_t v : g.neighbors(u)) {
                if (side[v] == side[u]) return {false, {}};
                if (side[v] == -1) {
                    side[v] = char(side[u] ^ 1);
                    order.push_back(v);
                }
            }
        }
    }
    return {true, std::move(side)};
}

}  // namespace saba
