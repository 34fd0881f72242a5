// Host graph builder, gradient-graph construction and compression pass.
// PAPER.md §2 :159-185 (graph), §4.1 :494-518 (gradients), §5.5 :813-821.
#include "graph.h"

#include <algorithm>
#include <map>
#include <string>
#include <cstdio>
#include <cstring>

#include "common.h"

namespace dflow {

const char* op_name(Op op) {
  switch (op) {
    case Op::Placeholder: return "Placeholder";
    case Op::Variable: return "Variable";
    case Op::MatMul: return "MatMul";
    case Op::Add: return "Add";
    case Op::Relu: return "Relu";
    case Op::Loss: return "Loss";
    case Op::LossGrad: return "LossGrad";
    case Op::ReluGrad: return "ReluGrad";
    case Op::ReduceSum: return "ReduceSum";
    case Op::AddN: return "AddN";
    case Op::ZerosLike: return "ZerosLike";
    case Op::ApplyGradientDescent: return "ApplyGradientDescent";
    case Op::Truncate16: return "Truncate16";
    case Op::CrossReplicaMeanT16: return "CrossReplicaMeanT16";
    case Op::Expand16: return "Expand16";
    case Op::CrossReplicaMean: return "CrossReplicaMean";
    case Op::StochasticRound16: return "StochasticRound16";
    case Op::CrossReplicaMeanSR16: return "CrossReplicaMeanSR16";
    case Op::Send: return "Send";
    case Op::Recv: return "Recv";
  }
  return "?";
}

static bool name_ok(const char* s) {
  if (!s || !*s) return false;
  for (const char* p = s; *p; ++p) {
    const char c = *p;
    if (!((c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || (c >= '0' && c <= '9') || c == '_' || c == '.' ||
          c == '/'))
      return false;
  }
  return true;
}

static bool dim_ok(int64_t a, int64_t b) { return a == b || a == DFLOW_BATCH || b == DFLOW_BATCH; }

dflow_status Graph::append(Node n, int* out) {
  if (!name_ok(n.name.c_str())) return fail(DFLOW_INVALID_ARGUMENT, "bad node name '%s'", n.name.c_str());
  if (by_name.count(n.name)) return fail(DFLOW_DUPLICATE_NAME, "duplicate node name '%s'", n.name.c_str());
  const int id = static_cast<int>(nodes.size());
  by_name.emplace(n.name, id);
  nodes.push_back(std::move(n));
  if (out) *out = id;
  return DFLOW_OK;
}

static dflow_status check_dtype(dflow_dtype dt) {
  if (dt != DFLOW_F32 && dt != DFLOW_BF16) return fail(DFLOW_INVALID_ARGUMENT, "dtype must be F32 or BF16");
  return DFLOW_OK;
}

dflow_status Graph::placeholder(const char* name, dflow_dtype dt, int rank, const int64_t* dims, int* out) {
  if (check_dtype(dt)) return DFLOW_INVALID_ARGUMENT;
  if (rank < 0 || rank > 2 || (rank > 0 && !dims)) return fail(DFLOW_INVALID_ARGUMENT, "placeholder rank must be 0..2");
  Node n;
  n.name = name ? name : "";
  n.op = Op::Placeholder;
  n.dtype = dt;
  for (int i = 0; i < rank; ++i) {
    if (dims[i] < 0 && dims[i] != DFLOW_BATCH) return fail(DFLOW_INVALID_ARGUMENT, "bad dim");
    n.shape.push_back(dims[i]);
  }
  return append(std::move(n), out);
}

dflow_status Graph::variable(const char* name, dflow_dtype dt, int rank, const int64_t* dims, int* out) {
  if (dt != DFLOW_F32) return fail(DFLOW_INVALID_ARGUMENT, "variables are fp32 (master weights, reading A13)");
  if (rank < 1 || rank > 2 || !dims) return fail(DFLOW_INVALID_ARGUMENT, "variable rank must be 1 or 2");
  Node n;
  n.name = name ? name : "";
  n.op = Op::Variable;
  n.dtype = dt;
  for (int i = 0; i < rank; ++i) {
    if (dims[i] <= 0) return fail(DFLOW_SHAPE_MISMATCH, "variables need static positive dims");
    n.shape.push_back(dims[i]);
  }
  return append(std::move(n), out);
}

dflow_status Graph::matmul(const char* name, int a, int b, int ta, int tb, int* out) {
  if (!valid(a) || !valid(b)) return fail(DFLOW_DANGLING_INPUT, "MatMul input does not exist");
  const Node &A = nodes[a], &B = nodes[b];
  if (A.shape.size() != 2 || B.shape.size() != 2) return fail(DFLOW_SHAPE_MISMATCH, "MatMul needs rank-2 inputs");
  const int64_t m = ta ? A.shape[1] : A.shape[0], ka = ta ? A.shape[0] : A.shape[1];
  const int64_t kb = tb ? B.shape[1] : B.shape[0], n = tb ? B.shape[0] : B.shape[1];
  if (!dim_ok(ka, kb))
    return fail(DFLOW_SHAPE_MISMATCH, "MatMul inner dims %lld vs %lld", (long long)ka, (long long)kb);
  Node nd;
  nd.name = name ? name : "";
  nd.op = Op::MatMul;
  nd.inputs = {a, b};
  nd.dtype = A.dtype;
  nd.shape = {m, n};
  nd.transpose_a = ta ? 1 : 0;
  nd.transpose_b = tb ? 1 : 0;
  return append(std::move(nd), out);
}

dflow_status Graph::add(const char* name, int a, int b, int* out) {
  if (!valid(a) || !valid(b)) return fail(DFLOW_DANGLING_INPUT, "Add input does not exist");
  const Node &A = nodes[a], &B = nodes[b];
  if (B.shape.size() == 1 && A.shape.size() == 2) {
    if (!dim_ok(A.shape[1], B.shape[0])) return fail(DFLOW_SHAPE_MISMATCH, "bias length mismatch");
  } else {
    bool ok = A.shape.size() == B.shape.size();
    for (size_t i = 0; ok && i < A.shape.size(); ++i) ok = dim_ok(A.shape[i], B.shape[i]);
    if (!ok) return fail(DFLOW_SHAPE_MISMATCH, "Add shapes are not compatible");
  }
  Node nd;
  nd.name = name ? name : "";
  nd.op = Op::Add;
  nd.inputs = {a, b};
  nd.dtype = A.dtype;
  nd.shape = A.shape;
  return append(std::move(nd), out);
}

dflow_status Graph::relu(const char* name, int x, int* out) {
  if (!valid(x)) return fail(DFLOW_DANGLING_INPUT, "Relu input does not exist");
  Node nd;
  nd.name = name ? name : "";
  nd.op = Op::Relu;
  nd.inputs = {x};
  nd.dtype = nodes[x].dtype;
  nd.shape = nodes[x].shape;
  return append(std::move(nd), out);
}

dflow_status Graph::loss(const char* name, int kind, int pred, int target, int* out) {
  if (kind != DFLOW_LOSS_MSE && kind != DFLOW_LOSS_SUM) return fail(DFLOW_INVALID_ARGUMENT, "unknown loss kind");
  if (!valid(pred)) return fail(DFLOW_DANGLING_INPUT, "loss prediction does not exist");
  const Node& P = nodes[pred];
  if (P.shape.size() != 2) return fail(DFLOW_SHAPE_MISMATCH, "loss needs a rank-2 prediction");
  Node nd;
  nd.name = name ? name : "";
  nd.op = Op::Loss;
  nd.inputs = {pred};
  nd.loss_kind = kind;
  nd.dtype = DFLOW_F32;
  if (kind == DFLOW_LOSS_MSE) {
    if (!valid(target)) return fail(target < 0 ? DFLOW_INVALID_ARGUMENT : DFLOW_DANGLING_INPUT, "MSE needs a target");
    const Node& T = nodes[target];
    if (T.shape.size() != 2 || !dim_ok(T.shape[0], P.shape[0]) || !dim_ok(T.shape[1], P.shape[1]))
      return fail(DFLOW_SHAPE_MISMATCH, "loss target shape mismatch");
    nd.inputs.push_back(target);
  } else if (target != -1) {
    return fail(DFLOW_INVALID_ARGUMENT, "SUM loss takes no target (pass -1)");
  }
  return append(std::move(nd), out);
}

dflow_status Graph::apply_gradient_descent(const char* name, int var, float lr, int grad, int* out) {
  if (!valid(var) || !valid(grad)) return fail(DFLOW_DANGLING_INPUT, "ApplyGradientDescent input does not exist");
  if (nodes[var].op != Op::Variable) return fail(DFLOW_INVALID_ARGUMENT, "ApplyGradientDescent needs a Variable");
  if (nodes[var].shape != nodes[grad].shape) return fail(DFLOW_SHAPE_MISMATCH, "gradient shape != variable shape");
  Node nd;
  nd.name = name ? name : "";
  nd.op = Op::ApplyGradientDescent;
  nd.inputs = {var, grad};
  nd.lr = lr;
  nd.dtype = DFLOW_F32;
  nd.shape = nodes[var].shape;
  return append(std::move(nd), out);
}

// ------------------------------------------------------------------ gradients
dflow_status Graph::gradients(int cost, const std::vector<int>& xs, std::vector<int>* out) {
  const std::vector<Node> saved_nodes = nodes;
  const auto saved_names = by_name;
  dflow_status st = gradients_impl(cost, xs, out);
  if (st != DFLOW_OK) {
    nodes = saved_nodes;
    by_name = saved_names;
  }
  return st;
}

dflow_status Graph::sum_partials(int node, const std::vector<int>& parts, int* out) {
  if (parts.empty()) return fail(DFLOW_NON_DIFFERENTIABLE, "no gradient reaches '%s'", nodes[node].name.c_str());
  if (parts.size() == 1) {
    *out = parts[0];
    return DFLOW_OK;
  }
  Node nd;
  nd.name = "grad/" + nodes[node].name + "/sum";
  nd.op = Op::AddN;
  nd.inputs = parts;
  nd.dtype = nodes[node].dtype;
  nd.shape = nodes[node].shape;
  return append(std::move(nd), out);
}

dflow_status Graph::gradient_function(int n, int g, const std::vector<char>& on_path,
                                      std::vector<std::pair<int, int>>* partials) {
  const Node fwd = nodes[n];  // copy: append() may reallocate `nodes`
  const std::string base = "grad/" + fwd.name + "/";
  int id = -1;
  dflow_status st;
  switch (fwd.op) {
    case Op::Loss: {
      const int pred = fwd.inputs[0];
      if (fwd.inputs.size() > 1 && on_path[fwd.inputs[1]])
        return fail(DFLOW_NON_DIFFERENTIABLE, "gradient with respect to the loss target of '%s'", fwd.name.c_str());
      if (on_path[pred]) {
        // dC/dpred with dC/dC = 1 folded in (the cost's registered gradient function)
        Node nd;
        nd.name = base + "pred";
        nd.op = Op::LossGrad;
        nd.inputs = fwd.inputs;
        nd.loss_kind = fwd.loss_kind;
        nd.dtype = nodes[pred].dtype;
        nd.shape = nodes[pred].shape;
        if ((st = append(std::move(nd), &id))) return st;
        partials->push_back({pred, id});
      }
      return DFLOW_OK;
    }
    case Op::Relu: {
      const int x = fwd.inputs[0];
      if (on_path[x]) {
        Node nd;  // ReluGrad(g, y): uses the forward OUTPUT y (a grey-arrow input)
        nd.name = base + "x";
        nd.op = Op::ReluGrad;
        nd.inputs = {g, n};
        nd.dtype = fwd.dtype;
        nd.shape = fwd.shape;
        if ((st = append(std::move(nd), &id))) return st;
        partials->push_back({x, id});
      }
      return DFLOW_OK;
    }
    case Op::Add: {
      const int a = fwd.inputs[0], b = fwd.inputs[1];
      if (on_path[a]) partials->push_back({a, g});  // identity partial
      if (on_path[b]) {
        if (nodes[b].shape.size() == 1 && nodes[a].shape.size() == 2) {
          Node nd;  // broadcast operand: sum the partial over the broadcast (row) axis
          nd.name = base + "b";
          nd.op = Op::ReduceSum;
          nd.inputs = {g};
          nd.axis = 0;
          nd.dtype = nodes[b].dtype;
          nd.shape = nodes[b].shape;
          if ((st = append(std::move(nd), &id))) return st;
          partials->push_back({b, id});
        } else {
          partials->push_back({b, g});
        }
      }
      return DFLOW_OK;
    }
    case Op::MatMul: {
      const int a = fwd.inputs[0], b = fwd.inputs[1];
      // C = op(A) op(B).  (ta,tb) -> dA = MatMul(x1, y1, t1a, t1b), dB = MatMul(x2, y2, t2a, t2b)
      struct R { int x, y, ta, tb; };
      R ra, rb;
      if (!fwd.transpose_a && !fwd.transpose_b) { ra = {g, b, 0, 1}; rb = {a, g, 1, 0}; }
      else if (fwd.transpose_a && !fwd.transpose_b) { ra = {b, g, 0, 1}; rb = {a, g, 0, 0}; }
      else if (!fwd.transpose_a && fwd.transpose_b) { ra = {g, b, 0, 0}; rb = {g, a, 1, 0}; }
      else { ra = {b, g, 1, 1}; rb = {g, a, 1, 1}; }
      if (on_path[a]) {
        if ((st = matmul((base + "a").c_str(), ra.x, ra.y, ra.ta, ra.tb, &id))) return st;
        partials->push_back({a, id});
      }
      if (on_path[b]) {
        if ((st = matmul((base + "b").c_str(), rb.x, rb.y, rb.ta, rb.tb, &id))) return st;
        partials->push_back({b, id});
      }
      return DFLOW_OK;
    }
    default:
      return fail(DFLOW_NON_DIFFERENTIABLE, "op %s ('%s') has no gradient function", op_name(fwd.op),
                  fwd.name.c_str());
  }
}

dflow_status Graph::gradients_impl(int cost, const std::vector<int>& xs, std::vector<int>* out) {
  if (!valid(cost)) return fail(DFLOW_DANGLING_INPUT, "cost node does not exist");
  for (int x : xs)
    if (!valid(x)) return fail(DFLOW_DANGLING_INPUT, "gradient source does not exist");
  if (!nodes[cost].shape.empty()) return fail(DFLOW_NON_SCALAR_TARGET, "cost '%s' is not scalar", nodes[cost].name.c_str());
  const int n0 = static_cast<int>(nodes.size());
  // 1. the path from the sources to C: reachable forward from some x and backward from C
  std::vector<char> fwd(n0, 0), back(n0, 0), on_path(n0, 0);
  for (int x : xs) fwd[x] = 1;
  for (int i = 0; i < n0; ++i)
    for (int in : nodes[i].inputs)
      if (fwd[in]) fwd[i] = 1;
  back[cost] = 1;
  for (int i = n0 - 1; i >= 0; --i)
    if (back[i])
      for (int in : nodes[i].inputs) back[in] = 1;
  for (int i = 0; i < n0; ++i) on_path[i] = fwd[i] && back[i];
  // 2. backtrack from C in reverse topological (= reverse construction) order
  std::vector<std::vector<int>> partials(n0);
  std::vector<int> total(n0, -1);
  std::vector<char> path_big;
  for (int i = n0 - 1; i >= 0; --i) {
    if (!on_path[i]) continue;
    int g = -1;
    dflow_status st;
    if (i != cost) {
      if ((st = sum_partials(i, partials[i], &g))) return st;
      total[i] = g;
    }
    if (nodes[i].op == Op::Placeholder || nodes[i].op == Op::Variable) continue;
    std::vector<std::pair<int, int>> p;
    path_big.assign(nodes.size(), 0);
    std::copy(on_path.begin(), on_path.end(), path_big.begin());
    if ((st = gradient_function(i, g, path_big, &p))) return st;
    for (auto& pr : p) partials[pr.first].push_back(pr.second);
  }
  out->clear();
  for (int x : xs) {
    if (x == cost) return fail(DFLOW_NON_DIFFERENTIABLE, "gradient of the cost with respect to itself");
    if (total[x] >= 0) {
      out->push_back(total[x]);
    } else if (on_path[x]) {
      int g;
      dflow_status st = sum_partials(x, partials[x], &g);
      if (st) return st;
      total[x] = g;
      out->push_back(g);
    } else {
      // C does not depend on x: zero partial
      Node nd;
      nd.name = "grad/" + nodes[x].name + "/zeros";
      nd.op = Op::ZerosLike;
      nd.inputs = {x};
      nd.dtype = nodes[x].dtype;
      nd.shape = nodes[x].shape;
      int id;
      dflow_status st = append(std::move(nd), &id);
      if (st) return st;
      total[x] = id;
      out->push_back(id);
    }
  }
  return DFLOW_OK;
}

// ------------------------------------------------------------------ JSON
static void json_str(std::string& o, const std::string& s) {
  o += '"';
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  o += '"';
}

static const char* dtype_str(dflow_dtype d) {
  switch (d) {
    case DFLOW_F32: return "f32";
    case DFLOW_BF16: return "bf16";
    case DFLOW_U16: return "u16";
  }
  return "?";
}

std::string Graph::to_json() const {
  std::string o = "{\"nodes\": [";
  char buf[64];
  for (size_t i = 0; i < nodes.size(); ++i) {
    const Node& n = nodes[i];
    if (i) o += ", ";
    o += "{\"attrs\": {";
    switch (n.op) {
      case Op::MatMul:
        snprintf(buf, sizeof buf, "\"transpose_a\": %d, \"transpose_b\": %d", n.transpose_a, n.transpose_b);
        o += buf;
        break;
      case Op::Loss:
      case Op::LossGrad:
        o += n.loss_kind == DFLOW_LOSS_MSE ? "\"kind\": \"MSE\"" : "\"kind\": \"SUM\"";
        break;
      case Op::ReduceSum:
        snprintf(buf, sizeof buf, "\"axis\": %d", n.axis);
        o += buf;
        break;
      case Op::ApplyGradientDescent:
        snprintf(buf, sizeof buf, "\"lr\": %.17g", static_cast<double>(n.lr));
        o += buf;
        break;
      case Op::CrossReplicaMean:
      case Op::CrossReplicaMeanT16:
      case Op::CrossReplicaMeanSR16:
        snprintf(buf, sizeof buf, "\"world\": %d", n.world);
        o += buf;
        break;
      case Op::Send:
      case Op::Recv:
        snprintf(buf, sizeof buf, "\"recv_device\": %d, \"send_device\": %d, \"tensor_name\": ", n.recv_device,
                 n.send_device);
        o += buf;
        json_str(o, n.tensor_name);
        break;
      default:
        break;
    }
    o += "}, \"dtype\": ";
    json_str(o, dtype_str(n.dtype));
    o += ", \"inputs\": [";
    for (size_t k = 0; k < n.inputs.size(); ++k) {
      if (k) o += ", ";
      json_str(o, nodes[n.inputs[k]].name);
    }
    o += "], \"name\": ";
    json_str(o, n.name);
    o += ", \"op\": ";
    json_str(o, op_name(n.op));
    o += ", \"shape\": [";
    for (size_t k = 0; k < n.shape.size(); ++k) {
      if (k) o += ", ";
      snprintf(buf, sizeof buf, "%lld", static_cast<long long>(n.shape[k]));
      o += buf;
    }
    o += "]}";
  }
  o += "], \"version\": 1}";
  return o;
}

// ------------------------------------------------------------------ exchange pass
dflow_status insert_exchange(const Graph& in, int world, int exchange, Graph* out, std::vector<int>* remap) {
  *out = Graph();
  remap->assign(in.nodes.size(), -1);
  // asynchronous replicas (f3): each replica's coded gradient goes straight to the apply
  const bool async = (exchange & DFLOW_EXCHANGE_ASYNC) != 0;
  exchange &= ~DFLOW_EXCHANGE_ASYNC;
  const bool active = world > 1 && exchange != DFLOW_EXCHANGE_NONE &&
                      !(async && (exchange == DFLOW_EXCHANGE_FP32 || exchange == DFLOW_EXCHANGE_FP32_NCCL));
  for (size_t i = 0; i < in.nodes.size(); ++i) {
    Node n = in.nodes[i];
    for (int& k : n.inputs) k = (*remap)[k];
    if (active && n.op == Op::ApplyGradientDescent) {
      const std::string var = in.nodes[in.nodes[i].inputs[0]].name;
      int g = n.inputs[1];
      const Node gnode = out->nodes[g];
      int id;
      dflow_status st;
      if (exchange == DFLOW_EXCHANGE_TRUNC16 || exchange == DFLOW_EXCHANGE_SR16) {
        const bool sr = exchange == DFLOW_EXCHANGE_SR16;
        Node t;
        t.name = "xchg/" + var + (sr ? "/sround16" : "/trunc16");
        t.op = sr ? Op::StochasticRound16 : Op::Truncate16;
        t.inputs = {g};
        t.dtype = DFLOW_U16;
        t.shape = gnode.shape;
        if ((st = out->append(t, &id))) return st;
        if (!async) {
          Node m;
          m.name = "xchg/" + var + "/mean";
          m.op = sr ? Op::CrossReplicaMeanSR16 : Op::CrossReplicaMeanT16;
          m.inputs = {id};
          m.dtype = DFLOW_U16;
          m.shape = gnode.shape;
          m.world = world;
          if ((st = out->append(m, &id))) return st;
        }
        Node e;
        e.name = "xchg/" + var + "/expand16";
        e.op = Op::Expand16;
        e.inputs = {id};
        e.dtype = DFLOW_F32;
        e.shape = gnode.shape;
        if ((st = out->append(e, &id))) return st;
      } else {
        Node m;
        m.name = "xchg/" + var + "/mean";
        m.op = Op::CrossReplicaMean;
        m.inputs = {g};
        m.dtype = DFLOW_F32;
        m.shape = gnode.shape;
        m.world = world;
        if ((st = out->append(m, &id))) return st;
      }
      n.inputs[1] = id;
    }
    int nid;
    dflow_status st = out->append(std::move(n), &nid);
    if (st) return st;
    (*remap)[i] = nid;
  }
  return DFLOW_OK;
}

// ------------------------------------------------------------------ partition pass (f4)
dflow_status partition(const Graph& in, const std::vector<int>& place, bool compress, std::vector<Graph>* out) {
  const int n = static_cast<int>(in.nodes.size());
  if (static_cast<int>(place.size()) != n) return fail(DFLOW_INVALID_ARGUMENT, "placement size != node count");
  int ndev = 0;
  for (int d : place) {
    if (d < 0) return fail(DFLOW_INVALID_ARGUMENT, "negative device in the placement");
    ndev = std::max(ndev, d + 1);
  }
  out->assign(ndev, Graph());
  std::vector<std::vector<int>> local(ndev, std::vector<int>(n, -1));
  std::map<std::pair<int, int>, int> chan;  // (endpoint, destination) -> node providing it there
  for (int i = 0; i < n; ++i) {
    const int d = place[i];
    Node nd = in.nodes[i];
    for (int& k : nd.inputs) {
      const int src = place[k];
      if (src == d) {
        k = local[d][k];
        continue;
      }
      auto it = chan.find({k, d});
      if (it == chan.end()) {
        const Node& x = in.nodes[k];
        const std::string key = x.name + "/" + std::to_string(src) + "to" + std::to_string(d);
        int id = local[src][k];
        dflow_status st;
        if (compress) {
          Node t;
          t.name = "chan/" + key + "/trunc16";
          t.op = Op::Truncate16;
          t.inputs = {id};
          t.dtype = DFLOW_U16;
          t.shape = x.shape;
          if ((st = (*out)[src].append(t, &id))) return st;
        }
        Node s;
        s.name = "send/" + key;
        s.op = Op::Send;
        s.inputs = {id};
        s.dtype = compress ? DFLOW_U16 : DFLOW_F32;
        s.shape = x.shape;
        s.tensor_name = x.name;
        s.send_device = src;
        s.recv_device = d;
        int sid;
        if ((st = (*out)[src].append(s, &sid))) return st;
        Node r = s;
        r.name = "recv/" + key;
        r.op = Op::Recv;
        r.inputs.clear();
        int rid;
        if ((st = (*out)[d].append(r, &rid))) return st;
        if (compress) {
          Node e;
          e.name = "chan/" + key + "/expand16";
          e.op = Op::Expand16;
          e.inputs = {rid};
          e.dtype = DFLOW_F32;
          e.shape = x.shape;
          if ((st = (*out)[d].append(e, &rid))) return st;
        }
        it = chan.emplace(std::make_pair(k, d), rid).first;
      }
      k = it->second;
    }
    int id;
    dflow_status st = (*out)[d].append(std::move(nd), &id);
    if (st) return st;
    local[d][i] = id;
  }
  return DFLOW_OK;
}

}  // namespace dflow
