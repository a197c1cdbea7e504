// Performance evaluator core (decider.hpp:46-94 of the reference), shared by
// the C-ABI (gnna_* in libgnna.so) and the gnnsim:: C++ drop-in.  Host code:
// the evaluator is scalar arithmetic over graph statistics.
#pragma once
#include <cstdint>
#include <vector>

#include "gnna.h"

namespace gnna_decider {

struct Grid {
    std::vector<uint32_t> gs, dw, tpb;
};

double alpha_from_degrees(double avg, double sd);
double wpt(const gnna_params& p);
uint64_t smem(const gnna_params& p);
uint32_t select_dw(uint32_t dim, uint32_t tpw);                 // throws gnna_decider::Domain
uint32_t select_ngs(uint32_t dw, uint32_t tpb, const gnna_model_inputs& in);
double dp_size(uint64_t smem_bytes, double avg);
double estimate_latency(const gnna_params& p, const gnna_model_inputs& in);
bool candidate_feasible(const gnna_params& p, const gnna_model_inputs& in);
bool feasibility(const gnna_params& p, const gnna_model_inputs& in);
gnna_params auto_params(const gnna_model_inputs& in);
void validate(const gnna_params& p);
struct SearchResult {
    gnna_params params;
    double latency;
    bool feasible;
    std::vector<double> trace;
};
SearchResult search_params(const gnna_model_inputs& in, uint32_t iterations, uint32_t population, uint64_t seed,
                           const Grid& grid);
gnna_model_inputs default_inputs();

struct Domain {
    const char* msg;
};

// B200 evaluator inputs: the graph's profile and the device's properties.
struct B200Inputs {
    uint64_t num_nodes = 0, num_edges = 0;
    uint32_t dim = 0, elem = 4;        // row width and element bytes (fp32 / fp64)
    uint64_t max_degree = 0;
    double l2_hit_share = 0.0;         // gather share of the top-degree rows that fit in L2/2 (x > L2)
    uint64_t window_bytes = 0;         // candidate L2 window (hub rows)
    double window_share = 0.0;         // gather share of the rows that fit in the window
    double window_rows_frac = 0.0;     // those rows / n
    uint32_t num_sms = 148;
    uint64_t l2_bytes = 0;
    double hbm_gbs = 0.0;
};
gnna_params b200_params(const B200Inputs& g, double* est_us, uint64_t* window_bytes);

}  // namespace gnna_decider
