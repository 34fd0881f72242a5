// Host dataflow-graph IR (§2 :159-185), gradient-graph construction
// (§4.1 :494-518) and the replicated-exchange compression pass
// (§5.5 :813-821 on the §7 :934-941 replica->combine transfer).
#pragma once
#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/dflow.h"

namespace dflow {

enum class Op : int {
  Placeholder,
  Variable,
  MatMul,
  Add,
  Relu,
  Loss,
  LossGrad,
  ReluGrad,
  ReduceSum,
  AddN,
  ZerosLike,
  ApplyGradientDescent,
  // inserted by insert_exchange (session graphs only)
  Truncate16,
  CrossReplicaMeanT16,
  Expand16,
  CrossReplicaMean,
  StochasticRound16,     // SR16 (f2)
  CrossReplicaMeanSR16,
  Send,                  // f4: cross-device channel endpoints
  Recv,
};

const char* op_name(Op op);

struct Node {
  std::string name;
  Op op;
  std::vector<int> inputs;
  dflow_dtype dtype = DFLOW_F32;
  std::vector<int64_t> shape;  // DFLOW_BATCH (-1) for the batch dimension
  int transpose_a = 0, transpose_b = 0;  // MatMul
  int loss_kind = -1;                     // Loss, LossGrad
  float lr = 0.f;                         // ApplyGradientDescent
  int axis = -1;                          // ReduceSum
  int world = 0;                          // exchange nodes
  std::string tensor_name;                // Send / Recv: the transferred endpoint
  int send_device = -1, recv_device = -1;  // Send / Recv
};

class Graph {
 public:
  std::vector<Node> nodes;
  std::unordered_map<std::string, int> by_name;

  dflow_status placeholder(const char* name, dflow_dtype dt, int rank, const int64_t* dims, int* out);
  dflow_status variable(const char* name, dflow_dtype dt, int rank, const int64_t* dims, int* out);
  dflow_status matmul(const char* name, int a, int b, int ta, int tb, int* out);
  dflow_status add(const char* name, int a, int b, int* out);
  dflow_status relu(const char* name, int x, int* out);
  dflow_status loss(const char* name, int kind, int pred, int target, int* out);
  dflow_status apply_gradient_descent(const char* name, int var, float lr, int grad, int* out);
  // Atomic: on failure the graph is restored.
  dflow_status gradients(int cost, const std::vector<int>& xs, std::vector<int>* out);

  std::string to_json() const;
  bool valid(int id) const { return id >= 0 && id < static_cast<int>(nodes.size()); }

  // Appends a fully-formed node after name validation (used by passes).
  dflow_status append(Node n, int* out);

 private:
  dflow_status gradients_impl(int cost, const std::vector<int>& xs, std::vector<int>* out);
  dflow_status sum_partials(int node, const std::vector<int>& parts, int* out);
  dflow_status gradient_function(int n, int g, const std::vector<char>& on_path,
                                 std::vector<std::pair<int, int>>* partials);
};

// Compression-insertion / replication pass (SPEC.md:681-689 shape).
// For world > 1, between every ApplyGradientDescent and its gradient input:
//   exchange TRUNC16: Truncate16 -> CrossReplicaMeanT16 -> Expand16
//   FP32 / FP32_NCCL: CrossReplicaMean
// world == 1 or exchange NONE: the graph is copied unchanged (reading A6).
// `remap[old_id] = new_id`.
dflow_status insert_exchange(const Graph& in, int world, int exchange, Graph* out, std::vector<int>* remap);

// Partition pass (f4): place[i] = device of node i.  Every cross-device
// edge x -> y becomes x -> [Truncate16 ->] Send in x's subgraph and Recv [-> Expand16] -> y
// in y's, one channel per (x, destination device) shared by all consumers there
// (canonicalisation); compress = the channel codec of PAPER.md:813-821.  out[d] = device
// d's subgraph, nodes in construction order.
dflow_status partition(const Graph& in, const std::vector<int>& place, bool compress, std::vector<Graph>* out);

}  // namespace dflow
