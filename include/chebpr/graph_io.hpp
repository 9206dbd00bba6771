// Drop-in for /root/reference/proj/include/chebpr/graph_io.hpp: edge-list and Matrix
// Market loaders feeding the K1 device builder.
#pragma once

#include <string>

#include "chebpr/graph.hpp"

namespace chebpr {

struct LoadOptions {
    bool dedup = true;
    bool drop_isolated = false;
    bool symmetrize = false;  // Matrix Market "general" files only
};

struct LoadedGraph {
    UndirectedGraph graph;
    GraphStats stats;
};

LoadedGraph load_edge_list(const std::string& path, const LoadOptions& opts = {});
LoadedGraph load_matrix_market(const std::string& path, const LoadOptions& opts = {});

}  // namespace chebpr
