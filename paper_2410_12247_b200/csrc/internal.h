// Internal declarations shared by the library's translation units.
#pragma once
#include <cstdint>
#include <string>

#include "../../include/epsmoe.h"

namespace epsmoe {

void set_error(const std::string& msg);
double cost_gemm_ms(const moe_cost_model_t& c, int kind, double m);
void default_cost_model(const moe_config_t& cfg, moe_cost_model_t* c);
int plan_slice_max(int e_loc, int64_t t_loc);
int default_comm_ctas();
double lr_rows_per_pair(int E, int D, int k, int N);
int plan_compute(const moe_config_t& cfg, const moe_cost_model_t& cost, int64_t global_tokens,
                 const int32_t* ghist, moe_plan_t* out);
int plan_normalise(const moe_config_t& cfg, moe_plan_t* p);

}  // namespace epsmoe
