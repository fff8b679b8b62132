#include "program.hpp"

#include <algorithm>
#include <cstdlib>
#include <map>
#include <set>
#include <sstream>
#include <tuple>
#include <unordered_map>
#include <unordered_set>

namespace planc_b200 {

const char* dtype_name(DType d) {
  switch (d) {
    case DType::f32: return "f32";
    case DType::bf16: return "bf16";
    case DType::i32: return "i32";
  }
  return "?";
}

const char* instr_kind_name(InstrKind k) {
  switch (k) {
    case InstrKind::gemm: return "gemm";
    case InstrKind::ew: return "ew";
    case InstrKind::reduce: return "reduce";
    case InstrKind::emb_lookup: return "emb_lookup";
    case InstrKind::emb_grad: return "emb_grad";
    case InstrKind::box: return "box";
    case InstrKind::xfer: return "xfer";
    case InstrKind::nop: return "nop";
    case InstrKind::rowwise: return "rowwise";
    case InstrKind::attention: return "attention";
  }
  return "?";
}

namespace {

std::vector<std::int64_t> row_major_strides(const std::vector<std::int64_t>& shape) {
  std::vector<std::int64_t> s(shape.size(), 1);
  for (int i = static_cast<int>(shape.size()) - 2; i >= 0; --i) s[i] = s[i + 1] * shape[i + 1];
  return s;
}

std::vector<std::int64_t> region_shape(const Region& r) {
  std::vector<std::int64_t> s;
  for (const auto& iv : r) s.push_back(iv.length());
  return s;
}

// Drops unit dims and merges dims that are contiguous in the destination and
// in every source term, so most cells become 1-D or 2-D strided copies.
void collapse(Cell& c) {
  int w = 0;
  for (int d = 0; d < c.rank; ++d) {
    if (c.extents[d] == 1) continue;
    c.extents[w] = c.extents[d];
    c.dst_strides[w] = c.dst_strides[d];
    for (auto& t : c.terms) t.strides[w] = t.strides[d];
    ++w;
  }
  c.rank = w;
  if (c.rank == 0) {
    c.rank = 1;
    c.extents[0] = 1;
    c.dst_strides[0] = 1;
    for (auto& t : c.terms) t.strides[0] = 1;
    return;
  }
  w = 0;
  for (int d = 1; d < c.rank; ++d) {
    bool ok = c.dst_strides[w] == c.dst_strides[d] * c.extents[d];
    for (const auto& t : c.terms) ok = ok && t.strides[w] == t.strides[d] * c.extents[d];
    if (ok) {
      c.extents[w] *= c.extents[d];
      c.dst_strides[w] = c.dst_strides[d];
      for (auto& t : c.terms) t.strides[w] = t.strides[d];
    } else {
      ++w;
      c.extents[w] = c.extents[d];
      c.dst_strides[w] = c.dst_strides[d];
      for (auto& t : c.terms) t.strides[w] = t.strides[d];
    }
  }
  c.rank = w + 1;
}

}  // namespace

std::vector<Cell> reconstruct_cells(const Mask& target, const std::vector<std::int64_t>& target_shape,
                                    const std::vector<std::pair<const Mask*, int>>& pieces,
                                    const std::vector<BufferDesc>& buffers, bool vv_extension,
                                    const std::string& ctx) {
  const Region& treg = target.region;
  const int rank = static_cast<int>(treg.size());
  if (rank > kMaxCellRank) throw UsageError("tensor rank above " + std::to_string(kMaxCellRank));
  struct Used {
    const Mask* mask;
    int buffer;
    bool add;
    bool part;  // V(m*v) -> V(v) sub-part (extension)
    Region ov;
  };
  std::vector<Used> used;
  std::int64_t touched = 0;
  for (const auto& [m, buf] : pieces) {
    bool add, part = false;
    if (m->value_count == target.value_count && m->value_index == target.value_index) {
      add = false;  // refexec.cpp:110-112 copy
    } else if (target.value_count == 1 && m->value_count > 1) {
      add = true;  // refexec.cpp:113-114 summand
    } else if (vv_extension && m->value_count > target.value_count &&
               m->value_count % target.value_count == 0 &&
               m->value_index / (m->value_count / target.value_count) == target.value_index) {
      add = part = true;  // V(m*v) -> V(v): sub-parts of the target's value part
    } else {
      continue;  // refexec.cpp:115-117
    }
    Region ov;
    if (!region_intersect(m->region, treg, &ov)) continue;
    touched += region_volume(ov);
    used.push_back({m, buf, add, part, ov});
  }
  if (touched < region_volume(treg)) {
    throw InternalError("reconstruct: region " + region_to_string(treg) + " not fully covered (" + ctx + ")");
  }
  // Grid of all overlap boundaries: inside each grid cell the ordered set of
  // contributing pieces is constant.
  std::vector<std::vector<std::int64_t>> bounds(rank);
  for (int d = 0; d < rank; ++d) {
    std::set<std::int64_t> b = {treg[d].lo, treg[d].hi};
    for (const auto& u : used) {
      b.insert(u.ov[d].lo);
      b.insert(u.ov[d].hi);
    }
    bounds[d].assign(b.begin(), b.end());
  }
  auto tstr = row_major_strides(target_shape);
  std::vector<Cell> cells;
  std::vector<std::size_t> idx(rank, 0);
  if (rank == 0) return cells;
  while (true) {
    Region box(rank);
    for (int d = 0; d < rank; ++d) box[d] = {bounds[d][idx[d]], bounds[d][idx[d] + 1]};
    Cell c;
    c.rank = rank;
    for (int d = 0; d < rank; ++d) {
      c.extents[d] = box[d].length();
      c.dst_strides[d] = tstr[d];
      c.dst_offset += (box[d].lo - treg[d].lo) * tstr[d];
    }
    // Sub-parts only fill cells no exact-match piece covers: where the
    // reference's copy rule applies its result stands and the sub-parts are
    // skipped (refexec.cpp:115-117), whatever the piece order.
    bool has_copy = false;
    for (const auto& u : used) {
      bool inside = true;
      for (int d = 0; d < rank; ++d) inside = inside && u.ov[d].lo <= box[d].lo && box[d].hi <= u.ov[d].hi;
      has_copy = has_copy || (inside && !u.add);
    }
    for (const auto& u : used) {
      bool inside = true;
      for (int d = 0; d < rank; ++d) inside = inside && u.ov[d].lo <= box[d].lo && box[d].hi <= u.ov[d].hi;
      if (!inside || (u.part && has_copy)) continue;
      const BufferDesc& src = buffers[u.buffer];
      auto sstr = row_major_strides(src.shape);
      Term t;
      t.buffer = u.buffer;
      t.add = u.add;
      for (int d = 0; d < rank; ++d) {
        t.strides[d] = sstr[d];
        t.offset += (box[d].lo - u.mask->region[d].lo) * sstr[d];
      }
      // A copy overwrites everything accumulated so far (refexec.cpp:126-130).
      if (!t.add) c.terms.clear();
      c.terms.push_back(t);
    }
    collapse(c);
    cells.push_back(std::move(c));
    int d = rank - 1;
    while (d >= 0) {
      if (++idx[d] + 1 < bounds[d].size()) break;
      idx[d] = 0;
      --d;
    }
    if (d < 0) break;
  }
  return cells;
}

namespace {

struct Builder {
  const ExecutionPlan& plan;
  const ProgramOptions& opt;
  Program P;
  std::map<int, int> lane_of_device;
  std::map<int, DType> pt_dtype;
  std::unordered_map<int, int> vt_buf;          // vt -> buffer
  std::map<std::tuple<int, int, std::vector<std::int64_t>>, int> placement;  // (lane, pt, region) -> buf
  std::unordered_set<int> issued_vts;
  std::unordered_map<int, int> channel_src;      // channel -> send input vt
  std::vector<int> op_last_instr;                // op idx -> last instruction (-1)
  std::vector<int> op_first_instr;
  std::unordered_map<int, std::vector<int>> sync_before;  // after op -> before ops
  std::vector<bool> op_issued;

  Builder(const ExecutionPlan& p, const ProgramOptions& o) : plan(p), opt(o) {}

  int lane_of_op(const OpNode& op) {
    auto it = plan.assignment.find(op.id);
    if (it == plan.assignment.end()) throw InternalError("op " + op.id + " has no device assignment");
    auto l = lane_of_device.find(it->second);
    if (l == lane_of_device.end()) {
      throw InternalError("op " + op.id + " assigned to device " + std::to_string(it->second) + " without a lane");
    }
    return l->second;
  }

  int new_buffer(int lane, int pt, const Mask& mask, int vt) {
    BufferDesc b;
    b.id = static_cast<int>(P.buffers.size());
    b.lane = lane;
    b.ptensor = pt;
    b.mask = mask;
    b.dtype = pt_dtype.at(pt);
    b.shape = region_shape(mask.region);
    b.elems = region_volume(mask.region);
    b.bytes = b.elems * dtype_size(b.dtype);
    b.vt = vt;
    std::int64_t& arena = P.lane_arena_bytes[lane];
    b.offset = arena;
    arena += (b.bytes + 255) / 256 * 256;
    P.buffers.push_back(b);
    return b.id;
  }

  int out_buffer(int vt_id, int lane) {
    const VTensor& v = plan.vt(vt_id);
    int b = new_buffer(lane, v.ptensor, v.mask, vt_id);
    vt_buf[vt_id] = b;
    if (static_cast<int>(P.vt_buffer.size()) <= vt_id) P.vt_buffer.resize(vt_id + 1, -1);
    P.vt_buffer[vt_id] = b;
    return b;
  }

  // refexec.cpp:378-394 (feed_ready / feed_value) + 366-376 (input_value)
  bool feed_ready(int cvt) {
    const VTensor& v = plan.vt(cvt);
    if (plan.is_graph_input(v.ptensor)) return true;
    auto f = plan.feeds.find(cvt);
    if (f == plan.feeds.end()) {
      throw InternalError("run_plan: consumer view " + std::to_string(cvt) + " of op " + v.owner_op +
                          " has no feed");
    }
    return issued_vts.count(f->second) > 0;
  }

  int input_buffer(int cvt, int lane) {
    auto f = plan.feeds.find(cvt);
    const VTensor& v = plan.vt(cvt);
    if (f != plan.feeds.end()) {
      int b = vt_buf.at(f->second);
      const BufferDesc& bd = P.buffers[b];
      if (!(bd.mask.region == v.mask.region)) {
        throw InternalError("feed of view " + std::to_string(cvt) + " covers " + region_to_string(bd.mask.region) +
                            ", consumer wants " + region_to_string(v.mask.region));
      }
      if (bd.lane != lane) {
        throw InternalError("feed of view " + std::to_string(cvt) + " crosses lanes without an adapter");
      }
      return b;
    }
    if (v.mask.value_count != 1) throw UsageError("run_plan: graph input consumed as partial value");
    std::vector<std::int64_t> key;
    for (const auto& iv : v.mask.region) {
      key.push_back(iv.lo);
      key.push_back(iv.hi);
    }
    auto k = std::make_tuple(lane, v.ptensor, key);
    auto it = placement.find(k);
    if (it != placement.end()) return it->second;
    Mask m;
    m.region = v.mask.region;
    int b = new_buffer(lane, v.ptensor, m, cvt);
    P.buffers[b].graph_input = true;
    TensorKind kind = plan.pt(v.ptensor).kind;
    P.buffers[b].weight = kind == TensorKind::weight || kind == TensorKind::optimizer_state;
    placement[k] = b;
    return b;
  }

  Instr& emit(InstrKind kind, int lane, int stream, int op_idx, const std::string& label) {
    Instr in;
    in.id = static_cast<int>(P.instrs.size());
    in.kind = kind;
    in.lane = lane;
    in.stream = stream;
    in.op = op_idx;
    in.label = label;
    P.instrs.push_back(std::move(in));
    P.issue_order.push_back(P.instrs.back().id);
    if (op_idx >= 0) {
      if (op_first_instr[op_idx] < 0) op_first_instr[op_idx] = P.instrs.back().id;
      op_last_instr[op_idx] = P.instrs.back().id;
    }
    return P.instrs.back();
  }

  void finish_deps(Instr& in) {
    std::set<int> d;
    for (int b : in.in_bufs) {
      if (P.buffers[b].producer >= 0) d.insert(P.buffers[b].producer);
    }
    for (const auto& c : in.cells) {
      for (const auto& t : c.terms) {
        if (P.buffers[t.buffer].producer >= 0) d.insert(P.buffers[t.buffer].producer);
      }
    }
    in.deps.assign(d.begin(), d.end());
    for (int b : in.out_bufs) P.buffers[b].producer = in.id;
  }

  double box_bytes(const Instr& in) {
    double by = 0;
    std::int64_t es = dtype_size(P.buffers[in.out_bufs[0]].dtype);
    for (const auto& c : in.cells) by += static_cast<double>(c.elems()) * es * (1 + c.terms.size());
    return by;
  }

  void emit_box(int op_idx, const OpNode& op, int lane, int stream, int out_vt,
                const std::vector<std::pair<const Mask*, int>>& pieces, const std::string& ctx) {
    int ob = out_buffer(out_vt, lane);
    const VTensor& ov = plan.vt(out_vt);
    Instr& in = emit(InstrKind::box, lane, stream, op_idx, op.id);
    in.out_bufs = {ob};
    in.cells = reconstruct_cells(ov.mask, P.buffers[ob].shape, pieces, P.buffers, opt.value_split_extension, ctx);
    std::set<int> ins;
    for (const auto& c : in.cells)
      for (const auto& t : c.terms) ins.insert(t.buffer);
    in.in_bufs.assign(ins.begin(), ins.end());
    in.bytes = box_bytes(in);
    finish_deps(in);
  }

  void exec_compute(int op_idx) {
    const OpNode& op = plan.ops[op_idx];
    int lane = lane_of_op(op);
    std::vector<int> ib;
    for (int v : op.inputs) ib.push_back(input_buffer(v, lane));
    auto shape_of = [&](int b) { return P.buffers[b].shape; };
    switch (op.kind) {
      case OpKind::matmul: {
        if (ib.size() != 2 || op.outputs.size() != 1) throw InternalError("matmul arity in " + op.id);
        auto a = shape_of(ib[0]), bsh = shape_of(ib[1]);
        if (a.size() != 2 || bsh.size() != 2) throw InternalError("matmul operands must be rank 2 in " + op.id);
        std::int64_t m = op.transpose_a ? a[1] : a[0], k = op.transpose_a ? a[0] : a[1];
        std::int64_t k2 = op.transpose_b ? bsh[1] : bsh[0], n = op.transpose_b ? bsh[0] : bsh[1];
        if (k != k2) throw InternalError("matmul operand inner extents differ in " + op.id);  // refexec.cpp:154
        int ob = out_buffer(op.outputs[0], lane);
        auto c = shape_of(ob);
        if (c.size() != 2 || c[0] != m || c[1] != n) throw InternalError("matmul output shape mismatch in " + op.id);
        Instr& in = emit(InstrKind::gemm, lane, 0, op_idx, op.id);
        in.in_bufs = ib;
        in.out_bufs = {ob};
        in.m = m;
        in.n = n;
        in.k = k;
        in.ta = op.transpose_a;
        in.tb = op.transpose_b;
        in.flops = 2.0 * m * n * k;
        in.bytes = static_cast<double>(P.buffers[ib[0]].bytes + P.buffers[ib[1]].bytes + P.buffers[ob].bytes);
        finish_deps(in);
        break;
      }
      case OpKind::ew_add:
      case OpKind::ew_mul:
      case OpKind::ew_max: {
        if (ib.empty() || op.outputs.size() != 1) throw InternalError("elementwise arity in " + op.id);
        for (std::size_t i = 1; i < ib.size(); ++i) {
          if (shape_of(ib[i]) != shape_of(ib[0])) throw InternalError("elementwise shape mismatch in " + op.id);
        }
        int ob = out_buffer(op.outputs[0], lane);
        if (P.buffers[ob].elems != P.buffers[ib[0]].elems) throw InternalError("elementwise output shape in " + op.id);
        Instr& in = emit(InstrKind::ew, lane, 0, op_idx, op.id);
        in.in_bufs = ib;
        in.out_bufs = {ob};
        in.ew = op.kind == OpKind::ew_add ? EwOp::add : op.kind == OpKind::ew_mul ? EwOp::mul : EwOp::max;
        in.count = P.buffers[ob].elems;
        in.flops = static_cast<double>(in.count) * (ib.size() - 1);
        in.bytes = static_cast<double>(in.count) * dtype_size(P.buffers[ob].dtype) * (ib.size() + 1);
        finish_deps(in);
        break;
      }
      case OpKind::reduce_sum: {
        if (ib.size() != 1 || op.outputs.size() != 1) throw InternalError("reduce arity in " + op.id);
        auto s = shape_of(ib[0]);
        int axis = op.axis < 0 ? 0 : op.axis;
        if (axis >= static_cast<int>(s.size())) throw InternalError("reduce axis out of range in " + op.id);
        int ob = out_buffer(op.outputs[0], lane);
        Instr& in = emit(InstrKind::reduce, lane, 0, op_idx, op.id);
        in.in_bufs = ib;
        in.out_bufs = {ob};
        in.outer = 1;
        in.inner = 1;
        for (int i = 0; i < axis; ++i) in.outer *= s[i];
        in.axis_len = s[axis];
        for (std::size_t i = axis + 1; i < s.size(); ++i) in.inner *= s[i];
        if (P.buffers[ob].elems != in.outer * in.inner) throw InternalError("reduce output shape in " + op.id);
        in.flops = static_cast<double>(P.buffers[ib[0]].elems);
        in.bytes = static_cast<double>(P.buffers[ib[0]].bytes + P.buffers[ob].bytes);
        finish_deps(in);
        break;
      }
      case OpKind::embedding_lookup: {
        if (ib.size() != 2 || op.outputs.size() != 1) throw InternalError("embedding arity in " + op.id);
        auto idx = shape_of(ib[0]), table = shape_of(ib[1]);
        if (idx.size() != 1 || table.size() != 2) throw InternalError("embedding operand ranks in " + op.id);
        int ob = out_buffer(op.outputs[0], lane);
        Instr& in = emit(InstrKind::emb_lookup, lane, 0, op_idx, op.id);
        in.in_bufs = ib;
        in.out_bufs = {ob};
        in.n_idx = idx[0];
        in.rows = table[0];
        in.h = table[1];
        in.lo = plan.vt(op.inputs[1]).mask.region[0].lo;  // refexec.cpp:219
        if (P.buffers[ob].elems != in.n_idx * in.h) throw InternalError("embedding output shape in " + op.id);
        std::int64_t es = dtype_size(P.buffers[ob].dtype);
        in.bytes = static_cast<double>(in.n_idx * 4 + 2 * in.n_idx * in.h * es);
        finish_deps(in);
        break;
      }
      case OpKind::embedding_grad: {
        if (ib.size() != 2 || op.outputs.size() != 1) throw InternalError("embedding-grad arity in " + op.id);
        auto idx = shape_of(ib[0]), g = shape_of(ib[1]);
        if (idx.size() != 1 || g.size() != 2) throw InternalError("embedding-grad operand ranks in " + op.id);
        int ob = out_buffer(op.outputs[0], lane);
        const Region& oreg = plan.vt(op.outputs[0]).mask.region;  // refexec.cpp:236-238
        Instr& in = emit(InstrKind::emb_grad, lane, 0, op_idx, op.id);
        in.in_bufs = ib;
        in.out_bufs = {ob};
        in.n_idx = idx[0];
        in.h = g[1];
        in.lo = oreg[0].lo;
        in.rows = oreg[0].length();
        if (P.buffers[ob].elems != in.rows * in.h) throw InternalError("embedding-grad output shape in " + op.id);
        std::int64_t es = dtype_size(P.buffers[ob].dtype);
        in.flops = static_cast<double>(in.n_idx * in.h);
        in.bytes = static_cast<double>(in.n_idx * 4 + in.n_idx * in.h * es + in.rows * in.h * es);
        finish_deps(in);
        break;
      }
      case OpKind::identity: {
        if (ib.size() != 1 || op.outputs.size() != 1) throw InternalError("identity arity in " + op.id);
        std::vector<std::pair<const Mask*, int>> pieces;
        Mask m = P.buffers[ib[0]].mask;
        const VTensor& ov = plan.vt(op.outputs[0]);
        // identity copies its operand whole (refexec.cpp:251): same extents,
        // placed at the output view's coordinates.
        if (region_shape(m.region) != region_shape(ov.mask.region)) {
          throw InternalError("identity shape mismatch in " + op.id);
        }
        Mask src = ov.mask;
        pieces.push_back({&src, ib[0]});
        emit_box(op_idx, op, lane, 0, op.outputs[0], pieces, "op " + op.id);
        P.instrs.back().label = op.id;
        break;
      }
      case OpKind::softmax:
      case OpKind::softmax_grad:
      case OpKind::layernorm:
      case OpKind::layernorm_grad:
      case OpKind::gelu:
      case OpKind::gelu_grad: {
        // Schema extension (oracle/planc_oracle.py eval_ext).
        const bool binary = op.kind == OpKind::softmax_grad || op.kind == OpKind::layernorm_grad ||
                            op.kind == OpKind::gelu_grad;
        if (ib.size() != (binary ? 2u : 1u) || op.outputs.size() != 1) throw InternalError("arity in " + op.id);
        int ob = out_buffer(op.outputs[0], lane);
        for (int b : ib)
          if (shape_of(b) != shape_of(ob)) throw InternalError("operand shape mismatch in " + op.id);
        Instr& in = emit(InstrKind::rowwise, lane, 0, op_idx, op.id);
        in.in_bufs = ib;
        in.out_bufs = {ob};
        in.count = P.buffers[ob].elems;
        in.row_op = op.kind == OpKind::softmax          ? RowOp::softmax
                    : op.kind == OpKind::softmax_grad   ? RowOp::softmax_grad
                    : op.kind == OpKind::layernorm      ? RowOp::layernorm
                    : op.kind == OpKind::layernorm_grad ? RowOp::layernorm_grad
                    : op.kind == OpKind::gelu           ? RowOp::gelu
                                                        : RowOp::gelu_grad;
        in.eps = op.eps;
        const auto sh = shape_of(ob);
        const std::int64_t n = sh.empty() ? 1 : sh.back();
        if (in.row_op != RowOp::gelu && in.row_op != RowOp::gelu_grad) {
          // Segments of the pTensor's last axis; a piece holds whole segments.
          const PTensor& pt = plan.pt(plan.vt(op.outputs[0]).ptensor);
          const std::int64_t full = pt.shape.empty() ? 1 : pt.shape.back();
          in.seg = op.segment > 0 ? op.segment : full;
          const Region& r = plan.vt(op.outputs[0]).mask.region;
          const std::int64_t lo = r.empty() ? 0 : r.back().lo;
          if (n % in.seg != 0 || lo % in.seg != 0 || full % in.seg != 0) {
            throw UsageError(std::string(op_kind_name(op.kind)) + " " + op.id +
                             ": the piece's last-axis region does not hold whole segments of " +
                             std::to_string(in.seg));
          }
          for (int v : op.inputs) {
            const Region& ri = plan.vt(v).mask.region;
            if (!ri.empty() && ri.back().lo % in.seg != 0) {
              throw UsageError(std::string(op_kind_name(op.kind)) + " " + op.id + ": input piece not segment-aligned");
            }
          }
        }
        const std::int64_t es = dtype_size(P.buffers[ob].dtype);
        in.bytes = static_cast<double>(in.count) * es * (ib.size() + 1);
        in.flops = static_cast<double>(in.count) * 8;
        finish_deps(in);
        break;
      }
      case OpKind::attention:
      case OpKind::attention_grad: {
        // Schema extension (oracle/planc_oracle.py eval_ext): a piece must
        // hold whole sequences and whole heads, and Q, K, V, O the same
        // region — a split inside a sequence or a head is rejected.
        const bool grad = op.kind == OpKind::attention_grad;
        if (ib.size() != (grad ? 5u : 3u) || op.outputs.size() != 1)
          throw InternalError(std::string(op_kind_name(op.kind)) + " arity in " + op.id);
        int ob = out_buffer(op.outputs[0], lane);
        const auto sh = shape_of(ob);
        for (int b : ib)
          if (shape_of(b) != sh) throw InternalError("attention operand shape mismatch in " + op.id);
        const Region& ro = plan.vt(op.outputs[0]).mask.region;
        for (int v : op.inputs) {
          if (!(plan.vt(v).mask.region == ro))
            throw UsageError("attention " + op.id + ": Q, K, V and O pieces must cover the same region");
        }
        if (sh.size() != 2 || op.head_dim <= 0 || op.seq <= 0)
          throw UsageError("attention " + op.id + ": needs rank-2 [tokens, heads x head_dim] tensors, head_dim and seq");
        if (ro[0].lo % op.seq != 0 || sh[0] % op.seq != 0 || ro[1].lo % op.head_dim != 0 || sh[1] % op.head_dim != 0)
          throw UsageError("attention " + op.id + ": the piece does not hold whole sequences of " +
                           std::to_string(op.seq) + " rows and whole heads of " + std::to_string(op.head_dim));
        const int wi = op.wrt == 'q' ? 0 : op.wrt == 'k' ? 1 : 2;
        if (grad) {
          // Join an earlier attention-grad instruction of this lane on the
          // same operands (dQ, dK, dV share the statistics pass and the
          // recomputed scores).
          for (auto it = P.instrs.rbegin(); it != P.instrs.rend(); ++it) {
            Instr& g = *it;
            if (g.kind != InstrKind::attention || g.att_grad == 0 || g.lane != lane || g.in_bufs != ib ||
                g.att_seq != op.seq || g.att_dh != op.head_dim || g.causal != op.causal || g.att_out[wi] >= 0)
              continue;
            g.att_out[wi] = ob;
            g.att_grad |= 1 << wi;
            g.out_bufs.push_back(ob);
            g.label += "+" + op.id;
            P.buffers[ob].producer = g.id;
            g.flops += (wi == 0 ? 1.0 : 0.5) * 4.0 * static_cast<double>(sh[0]) * static_cast<double>(op.seq) *
                       static_cast<double>(sh[1]) * (op.causal ? 0.5 : 1.0);
            g.bytes += static_cast<double>(sh[0] * sh[1]) * dtype_size(P.buffers[ob].dtype);
            ob = -1;
            break;
          }
          if (ob < 0) break;  // joined
        }
        Instr& in = emit(InstrKind::attention, lane, 0, op_idx, op.id);
        in.in_bufs = ib;
        in.out_bufs = {ob};
        if (grad) {
          in.att_grad = 1 << wi;
          in.att_out[wi] = ob;
        }
        in.att_rows = sh[0];
        in.att_cols = sh[1];
        in.att_seq = op.seq;
        in.att_dh = op.head_dim;
        in.causal = op.causal;
        const std::int64_t es = dtype_size(P.buffers[ob].dtype);
        in.bytes = static_cast<double>(sh[0] * sh[1]) * es * (grad ? 6 : 4);
        // forward: QK^T and PV per (sequence, head): 4 * seq^2 * dh (half with a
        // causal mask). Gradient (algorithmic, no recomputed scores): dP and
        // dQ for wrt = q (one forward's worth), dK or dV (half each) — 2x the
        // forward for all three.
        in.flops = (grad && wi > 0 ? 0.5 : 1.0) * 4.0 * static_cast<double>(sh[0]) * static_cast<double>(op.seq) *
                   static_cast<double>(sh[1]) * (op.causal ? 0.5 : 1.0);
        finish_deps(in);
        break;
      }
      default:
        throw UsageError(std::string("refexec: unsupported op kind ") + op_kind_name(op.kind) + " (" + op.id + ")");
    }
  }

  void exec_op(int op_idx) {
    const OpNode& op = plan.ops[op_idx];
    int lane = lane_of_op(op);
    switch (op.kind) {
      case OpKind::free_buffer:
        break;  // refexec.cpp:416-417: bookkeeping only
      case OpKind::send:
        if (op.inputs.size() != 1) throw InternalError("send arity in " + op.id);
        input_buffer(op.inputs[0], lane);
        channel_src[op.channel] = op.inputs[0];
        break;
      case OpKind::recv: {  // refexec.cpp:422-425
        if (op.outputs.size() != 1) throw InternalError("recv arity in " + op.id);
        int svt = channel_src.at(op.channel);
        const VTensor& sv = plan.vt(svt);
        int src_lane = lane_of_op(plan.op(sv.owner_op));
        int sb = input_buffer(svt, src_lane);
        const VTensor& ov = plan.vt(op.outputs[0]);
        if (region_shape(sv.mask.region) != region_shape(ov.mask.region)) {
          throw InternalError("channel " + std::to_string(op.channel) + " piece shape mismatch at " + op.id);
        }
        Mask src = ov.mask;  // the channel carries the value as-is
        std::vector<std::pair<const Mask*, int>> pieces = {{&src, sb}};
        emit_box(op_idx, op, lane, 1, op.outputs[0], pieces, "op " + op.id);
        Instr& in = P.instrs.back();
        in.wire_bytes = static_cast<double>(P.buffers[sb].bytes);
        break;
      }
      case OpKind::split:
      case OpKind::concat:
      case OpKind::reduce_assemble: {  // refexec.cpp:426-441
        std::vector<std::pair<const Mask*, int>> pieces;
        for (int v : op.inputs) pieces.push_back({&plan.vt(v).mask, input_buffer(v, lane)});
        for (int out : op.outputs) emit_box(op_idx, op, lane, 0, out, pieces, "op " + op.id);
        break;
      }
      default:
        exec_compute(op_idx);
    }
    for (int v : op.outputs) issued_vts.insert(v);
  }

  // refexec.cpp:459-481: every member's output reconstructed from all
  // members' input pieces.
  void exec_collective(const CollectiveGroup& grp) {
    std::vector<std::pair<const Mask*, int>> pieces;
    for (const auto& oid : grp.ops) {
      const OpNode& m = plan.op(oid);
      int lane = lane_of_op(m);
      for (int v : m.inputs) pieces.push_back({&plan.vt(v).mask, input_buffer(v, lane)});
    }
    double n = static_cast<double>(grp.message_bytes), k = grp.k;
    double wire = 0;  // NCCL bus-bandwidth conventions
    if (grp.primitive == "all-reduce") wire = 2.0 * (k - 1) / k * n;
    else if (grp.primitive == "all-gather" || grp.primitive == "reduce-scatter" || grp.primitive == "all-to-all")
      wire = (k - 1) / k * n;
    else wire = n;
    for (const auto& oid : grp.ops) {
      int oi = plan.op_idx(oid);
      const OpNode& m = plan.ops[oi];
      int lane = lane_of_op(m);
      for (int out : m.outputs) {
        emit_box(oi, m, lane, 1, out, pieces, "collective " + oid);
        P.instrs.back().wire_bytes = wire;
        P.instrs.back().label = grp.primitive + ":" + oid;
        P.instrs.back().coll_group = grp.id;
      }
      for (int v : m.outputs) issued_vts.insert(v);
      op_issued[oi] = true;
    }
  }

  bool sync_ready(int op_idx) {
    if (!opt.honor_sync_edges) return true;
    auto it = sync_before.find(op_idx);
    if (it == sync_before.end()) return true;
    for (int b : it->second) {
      if (!op_issued[b]) return false;
    }
    return true;
  }

  void add_sync_deps(int op_idx) {
    if (!opt.honor_sync_edges) return;
    auto it = sync_before.find(op_idx);
    if (it == sync_before.end() || op_first_instr[op_idx] < 0) return;
    Instr& first = P.instrs[op_first_instr[op_idx]];
    for (int b : it->second) {
      int li = op_last_instr[b];
      if (li >= 0 && P.instrs[li].lane != first.lane) {
        first.deps.push_back(li);
      }
    }
    std::sort(first.deps.begin(), first.deps.end());
    first.deps.erase(std::unique(first.deps.begin(), first.deps.end()), first.deps.end());
  }

  void run() {
    P.num_lanes = static_cast<int>(plan.lanes.size());
    P.lane_arena_bytes.assign(P.num_lanes, 0);
    for (int l = 0; l < P.num_lanes; ++l) {
      lane_of_device[plan.lanes[l].device] = l;
      P.lane_device.push_back(plan.lanes[l].device);
    }
    // Element types: elem_size 4 -> f32, 2 -> bf16; embedding index operands
    // hold integer row ids and are stored as i32 (refexec.cpp:221).
    std::set<int> index_pts;
    for (const auto& op : plan.ops) {
      if ((op.kind == OpKind::embedding_lookup || op.kind == OpKind::embedding_grad) && !op.inputs.empty()) {
        index_pts.insert(plan.vt(op.inputs[0]).ptensor);
      }
    }
    for (const auto& [id, pt] : plan.ptensors) {
      if (index_pts.count(id)) pt_dtype[id] = DType::i32;
      else if (pt.elem_size == 4) pt_dtype[id] = DType::f32;
      else if (pt.elem_size == 2) pt_dtype[id] = DType::bf16;
      else throw UsageError("unsupported elem_size " + std::to_string(pt.elem_size) + " on ptensor " +
                            std::to_string(id));
    }
    for (const auto& op : plan.ops) {
      if (op.kind == OpKind::embedding_lookup || op.kind == OpKind::embedding_grad || op.kind == OpKind::send ||
          op.kind == OpKind::recv || op.kind == OpKind::split || op.kind == OpKind::concat ||
          op.kind == OpKind::collective || op.kind == OpKind::free_buffer || op.kind == OpKind::identity) {
        continue;
      }
      for (int v : op.inputs) {
        if (index_pts.count(plan.vt(v).ptensor)) {
          throw UsageError("index tensor " + std::to_string(plan.vt(v).ptensor) + " consumed by " + op.id);
        }
      }
    }
    op_last_instr.assign(plan.ops.size(), -1);
    op_first_instr.assign(plan.ops.size(), -1);
    op_issued.assign(plan.ops.size(), false);
    for (const auto& [a, b] : plan.sync_edges) {
      sync_before[plan.op_idx(b)].push_back(plan.op_idx(a));
    }

    // Issue simulation: refexec.cpp:396-530 with "issued" as readiness.
    std::map<int, std::vector<int>> members;  // group -> op idx
    for (const auto& [gid, grp] : plan.coll_groups) {
      for (const auto& oid : grp.ops) members[gid].push_back(plan.op_idx(oid));
    }
    std::vector<std::size_t> cursor(P.num_lanes, 0);
    std::unordered_map<int, std::pair<int, std::size_t>> op_pos;
    std::vector<std::vector<int>> lane_ops(P.num_lanes);
    for (int l = 0; l < P.num_lanes; ++l) {
      for (std::size_t t = 0; t < plan.lanes[l].tasks.size(); ++t) {
        int oi = plan.op_idx(plan.lanes[l].tasks[t].op);
        op_pos[oi] = {l, t};
        lane_ops[l].push_back(oi);
      }
    }
    auto arrived = [&](int oi) {
      auto it = op_pos.find(oi);
      if (it == op_pos.end()) throw InternalError("collective member " + plan.ops[oi].id + " is in no lane");
      return cursor[it->second.first] == it->second.second;
    };
    std::set<int> channels_sent;
    bool progress = true;
    while (progress) {
      progress = false;
      for (int l = 0; l < P.num_lanes; ++l) {
        while (cursor[l] < lane_ops[l].size()) {
          int oi = lane_ops[l][cursor[l]];
          const OpNode& op = plan.ops[oi];
          bool ready = true;
          if (op.kind == OpKind::recv) {
            ready = channels_sent.count(op.channel) > 0;
          } else if (op.kind == OpKind::collective) {
            auto mit = members.find(op.coll_group);
            if (mit == members.end()) throw InternalError("unknown collective group for " + op.id);
            for (int m : mit->second) ready = ready && arrived(m);
            if (ready) {
              for (int m : mit->second)
                for (int v : plan.ops[m].inputs) ready = ready && feed_ready(v);
            }
            if (ready) {
              for (int m : mit->second) ready = ready && sync_ready(m);
            }
          } else {
            for (int v : op.inputs) ready = ready && feed_ready(v);
            ready = ready && sync_ready(oi);
          }
          if (!ready) break;
          if (op.kind == OpKind::collective) {
            exec_collective(plan.coll_groups.at(op.coll_group));
            for (int m : members.at(op.coll_group)) {
              add_sync_deps(m);
              auto [ml, mt] = op_pos.at(m);
              cursor[ml] = mt + 1;
            }
          } else {
            exec_op(oi);
            if (op.kind == OpKind::send) channels_sent.insert(op.channel);
            op_issued[oi] = true;
            add_sync_deps(oi);
            cursor[l]++;
          }
          progress = true;
        }
      }
    }
    for (int l = 0; l < P.num_lanes; ++l) {
      if (cursor[l] < lane_ops[l].size()) {
        throw InternalError("run_plan: pairing deadlock at task " + plan.ops[lane_ops[l][cursor[l]]].id +
                            " on device " + std::to_string(plan.lanes[l].device));
      }
    }

    // Output reassembly table (refexec.cpp:532-556).
    std::map<int, std::vector<int>> piece_vts;
    for (const auto& op : plan.ops) {
      if (op.inserted) continue;
      for (int v : op.outputs) piece_vts[plan.vt(v).ptensor].push_back(v);
    }
    for (const auto& [pt, vts] : piece_vts) {
      std::set<std::tuple<std::vector<std::int64_t>, int, int>> seen;
      std::vector<int> bufs;
      for (int v : vts) {
        const Mask& m = plan.vt(v).mask;
        std::vector<std::int64_t> key;
        for (const auto& iv : m.region) {
          key.push_back(iv.lo);
          key.push_back(iv.hi);
        }
        if (!seen.insert({key, m.value_index, m.value_count}).second) continue;
        auto it = vt_buf.find(v);
        if (it == vt_buf.end()) throw InternalError("output view " + std::to_string(v) + " was never produced");
        bufs.push_back(it->second);
      }
      P.outputs.push_back({pt, bufs});
    }
    std::set<int> gi;
    for (const auto& b : P.buffers) {
      if (b.graph_input) gi.insert(b.ptensor);
    }
    P.graph_inputs.assign(gi.begin(), gi.end());
    P.lane_flops.assign(P.num_lanes, 0);
    P.lane_bytes.assign(P.num_lanes, 0);
    P.lane_wire_bytes.assign(P.num_lanes, 0);
    for (const auto& in : P.instrs) {
      P.lane_flops[in.lane] += in.flops;
      P.lane_bytes[in.lane] += in.kind == InstrKind::gemm ? 0 : in.bytes;
      P.lane_wire_bytes[in.lane] += in.wire_bytes;
      P.total_flops += in.flops;
      P.total_bytes += in.kind == InstrKind::gemm ? 0 : in.bytes;
      P.total_wire_bytes += in.wire_bytes;
    }
  }
};

}  // namespace

Program build_program(const ExecutionPlan& plan, const ProgramOptions& opt) {
  Builder b(plan, opt);
  b.run();
  if (opt.two_phase_allreduce) two_phase_allreduce(b.P, opt);
  if (opt.fuse_epilogues) fuse_gemm_epilogues(b.P, opt);
  if (opt.fuse_epilogues && opt.fuse_box_ew) fuse_box_elementwise(b.P, opt);
  if (opt.gather_operands && opt.gemm_groupable) gather_gemm_operands(b.P, opt);
  if (opt.group_gemms && opt.gemm_groupable) group_gemms(b.P, opt);
  return std::move(b.P);
}

void group_gemms(Program& P, const ProgramOptions& opt) {
  const int n = static_cast<int>(P.instrs.size());
  std::vector<int> redirect(n, -1);  // grouped member -> its group's instruction
  auto red = [&](int d) { return redirect[d] >= 0 ? redirect[d] : d; };
  auto deps_of = [&](int x) {
    std::set<int> d;
    for (int y : P.instrs[x].deps) d.insert(red(y));
    d.erase(x);
    return d;
  };
  // Transitive ancestors (through redirected edges), sorted.
  std::vector<int> mark(n, -1);
  int stamp = 0;
  auto ancestors = [&](int x) {
    std::vector<int> anc, stack{x};
    ++stamp;
    while (!stack.empty()) {
      const int y = stack.back();
      stack.pop_back();
      for (int d0 : P.instrs[y].deps) {
        const int d = red(d0);
        if (d == y || mark[d] == stamp) continue;
        mark[d] = stamp;
        anc.push_back(d);
        stack.push_back(d);
      }
    }
    std::sort(anc.begin(), anc.end());
    return anc;
  };
  auto has = [](const std::vector<int>& v, int x) { return std::binary_search(v.begin(), v.end(), x); };
  struct Open {
    int leader;
    std::vector<int> anc;  // ancestors of the group (all members'), sorted
    std::set<int> deps;    // direct dependencies of the group
  };
  std::map<std::tuple<int, std::int64_t, std::int64_t, std::int64_t, bool, bool, int, int, int>, std::vector<Open>>
      open;
  constexpr std::size_t kWindow = 256;  // issue-order distance a group may span
  std::vector<int> pos(n, 0);
  for (std::size_t i = 0; i < P.issue_order.size(); ++i) pos[P.issue_order[i]] = static_cast<int>(i);
  for (int id : P.issue_order) {
    Instr& g = P.instrs[id];
    // Reduce-scatter GEMMs (scatter > 0) carry k receive slices as their
    // outputs: a grouped launch holds one output per member, so they never join.
    if (g.kind != InstrKind::gemm || !g.fused.empty() || g.group != 1 || g.scatter > 0 || !g.gather[0].empty() ||
        !g.gather[1].empty())
      continue;
    const DType da = P.buffers[g.in_bufs[0]].dtype, db = P.buffers[g.in_bufs[1]].dtype,
                dc = P.buffers[g.out_bufs[0]].dtype;
    if (!opt.gemm_groupable(g, da, db, dc)) continue;
    auto key = std::make_tuple(g.lane, g.m, g.n, g.k, g.ta, g.tb, static_cast<int>(da), static_cast<int>(db),
                               static_cast<int>(dc));
    const std::set<int> gd = deps_of(id);
    auto& cands = open[key];
    cands.erase(std::remove_if(cands.begin(), cands.end(),
                               [&](const Open& o) {
                                 return P.instrs[o.leader].group >= kMaxGemmGroupInstr ||
                                        pos[id] - pos[o.leader] > static_cast<int>(kWindow);
                               }),
                cands.end());
    const std::vector<int> ga = cands.empty() ? std::vector<int>{} : ancestors(id);
    bool joined = false;
    for (auto& o : cands) {
      Instr& L = P.instrs[o.leader];
      // Same readiness and independence: each side's dependencies are
      // ancestors of the other (so neither waits longer in the group, and
      // the group's slot in the issue order — the leader's — follows every
      // member's producers); the newcomer depends on no member.
      bool ok = !has(ga, o.leader);
      for (int d : gd) ok = ok && has(o.anc, d);
      for (int d : o.deps) ok = ok && has(ga, d);
      if (!ok) continue;
      L.in_bufs.push_back(g.in_bufs[0]);
      L.in_bufs.push_back(g.in_bufs[1]);
      L.out_bufs.push_back(g.out_bufs[0]);
      L.group += 1;
      L.flops += g.flops;
      L.bytes += g.bytes;
      L.label += "+" + g.label;
      P.buffers[g.out_bufs[0]].producer = o.leader;
      redirect[id] = o.leader;
      g.kind = InstrKind::nop;
      g.deps.clear();
      g.in_bufs.clear();
      g.out_bufs.clear();
      g.flops = g.bytes = 0;
      joined = true;
      break;
    }
    if (!joined) cands.push_back(Open{id, cands.empty() ? ancestors(id) : ga, gd});
  }
  for (auto& in : P.instrs) {
    bool changed = false;
    for (int& d : in.deps) {
      if (redirect[d] >= 0) {
        d = redirect[d];
        changed = true;
      }
    }
    if (changed) {
      std::sort(in.deps.begin(), in.deps.end());
      in.deps.erase(std::unique(in.deps.begin(), in.deps.end()), in.deps.end());
      in.deps.erase(std::remove(in.deps.begin(), in.deps.end(), in.id), in.deps.end());
    }
  }
}

void gather_gemm_operands(Program& P, const ProgramOptions& opt) {
  const int nb = static_cast<int>(P.buffers.size());
  std::vector<std::vector<int>> readers(nb);
  for (const auto& in : P.instrs) {
    if (in.kind == InstrKind::nop) continue;
    std::set<int> r;
    for (int b : in.in_bufs) r.insert(b);
    for (const auto& c : in.cells)
      for (const auto& t : c.terms) r.insert(t.buffer);
    for (const auto& fe : in.fused)
      for (int b : fe.in_bufs) r.insert(b);
    for (const auto& x : in.xfers) r.insert(x.src);
    for (int b : r) readers[b].push_back(in.id);
  }
  std::set<int> outputs;
  for (const auto& o : P.outputs)
    for (int b : o.second) outputs.insert(b);
  // Piece rows must be whole multiples of every TMA box height the GEMM may
  // load (BM = 128 rows, BK = 64 k-rows, BN <= 256 columns-as-rows).
  constexpr std::int64_t kPieceRowAlign = 256;
  for (auto& bx : P.instrs) {
    if (bx.kind != InstrKind::box || bx.out_bufs.size() != 1 || bx.cells.empty() ||
        bx.cells.size() > static_cast<std::size_t>(kMaxGemmGroupInstr))
      continue;
    const int O = bx.out_bufs[0];
    const BufferDesc& ob = P.buffers[O];
    if (ob.shape.size() != 2 || ob.graph_input || outputs.count(O) || ob.dtype != DType::bf16) continue;
    const std::int64_t R = ob.shape[0], C = ob.shape[1];
    // Cells: whole row blocks (or whole column blocks), one plain copy of a
    // dense piece each.
    std::vector<std::pair<std::int64_t, int>> pieces;  // (first row / column, source buffer)
    bool ok = true, by_cols = false;
    std::int64_t rows = -1, cols = -1;
    for (const auto& c : bx.cells) {
      if (c.terms.size() != 1 || c.terms[0].add || c.terms[0].fold >= 0 || c.terms[0].offset != 0) {
        ok = false;
        break;
      }
      const Term& t = c.terms[0];
      const BufferDesc& sb = P.buffers[t.buffer];
      const std::int64_t e = c.elems();
      if (sb.elems != e || sb.dtype != ob.dtype || sb.dead) {
        ok = false;
        break;
      }
      bool dense_rows = false, dense_cols = false;
      if (c.rank == 1) dense_rows = c.dst_strides[0] == 1 && t.strides[0] == 1 && e % C == 0 && c.dst_offset % C == 0;
      if (c.rank == 2) {
        dense_rows = c.extents[1] == C && c.dst_strides[0] == C && c.dst_strides[1] == 1 && t.strides[0] == C &&
                     t.strides[1] == 1 && c.dst_offset % C == 0;
        // a column block: all R rows, extents[1] columns starting at dst_offset
        dense_cols = c.extents[0] == R && c.extents[1] < C && c.dst_strides[0] == C && c.dst_strides[1] == 1 &&
                     t.strides[0] == c.extents[1] && t.strides[1] == 1 && c.dst_offset < C;
      }
      if (pieces.empty()) by_cols = dense_cols && !dense_rows;
      if (by_cols ? !dense_cols : !dense_rows) {
        ok = false;
        break;
      }
      if (by_cols) {
        if (cols < 0) cols = c.extents[1];
        ok = ok && c.extents[1] == cols;
        pieces.push_back({c.dst_offset, t.buffer});
      } else {
        if (rows < 0) rows = e / C;
        ok = ok && e / C == rows;
        pieces.push_back({c.dst_offset / C, t.buffer});
      }
    }
    // Piece columns: whole 64-element TMA boxes (a box never straddles two
    // pieces along the stored inner dimension).
    constexpr std::int64_t kPieceColAlign = 64;
    if (!ok || pieces.empty() || (by_cols && !opt.gather_cols)) continue;
    if (by_cols ? (cols <= 0 || cols % kPieceColAlign != 0 || static_cast<std::int64_t>(pieces.size()) * cols != C)
                : (rows <= 0 || rows % kPieceRowAlign != 0 || static_cast<std::int64_t>(pieces.size()) * rows != R))
      continue;
    std::sort(pieces.begin(), pieces.end());
    const std::int64_t ext = by_cols ? cols : rows;
    for (std::size_t i = 0; i < pieces.size(); ++i) ok = ok && pieces[i].first == static_cast<std::int64_t>(i) * ext;
    // Readers: tensor-core GEMMs only, O as one plain operand.
    std::vector<std::pair<int, int>> uses;  // (gemm, operand index)
    for (int r : readers[O]) {
      const Instr& g = P.instrs[r];
      const bool gem = g.kind == InstrKind::gemm && g.group == 1 && g.scatter == 0 && g.in_bufs.size() == 2 &&
                       (g.in_bufs[0] == O) != (g.in_bufs[1] == O);
      bool fused_reads = false;
      for (const auto& fe : g.fused)
        for (int b : fe.in_bufs) fused_reads = fused_reads || b == O;
      if (!ok || !gem || fused_reads || g.lane != bx.lane ||
          !opt.gemm_groupable(g, P.buffers[g.in_bufs[0]].dtype, P.buffers[g.in_bufs[1]].dtype,
                              P.buffers[g.out_bufs[0]].dtype)) {
        ok = false;
        break;
      }
      const int j = g.in_bufs[0] == O ? 0 : 1;
      // Column pieces only along K (A stored [m][k], B stored [n][k]): the
      // piece then changes every cols / BK k-blocks. Along M or N every
      // k-block's boxes alternate between the pieces' tensor maps, which
      // measured ~1.8x slower on C5's 2-SM dW GEMMs (TMA descriptor
      // switches; profiles/r02/ab_col_gather.jsonl).
      if (by_cols && (j == 0 ? g.ta : !g.tb)) {
        ok = false;
        break;
      }
      uses.push_back({r, j});
    }
    if (!ok || uses.empty()) continue;
    for (auto [r, j] : uses) {
      Instr& g = P.instrs[r];
      for (const auto& pc : pieces) g.gather[j].push_back(pc.second);
      g.gather_rows[j] = by_cols ? 0 : rows;
      g.gather_cols[j] = by_cols ? cols : 0;
      g.in_bufs[j] = pieces[0].second;  // (O is dead: never written nor read)
      // The GEMM waits for the pieces' producers (bx's dependencies).
      for (int d : bx.deps) g.deps.push_back(d);
      g.deps.erase(std::remove(g.deps.begin(), g.deps.end(), bx.id), g.deps.end());
      std::sort(g.deps.begin(), g.deps.end());
      g.deps.erase(std::unique(g.deps.begin(), g.deps.end()), g.deps.end());
      g.label += "<gather:" + bx.label + ">";
    }
    // bx stays as a nop (its deps still order anything a sync edge hangs on it).
    bx.kind = InstrKind::nop;
    bx.cells.clear();
    bx.out_bufs.clear();
    bx.bytes = 0;
    P.buffers[O].dead = true;
    P.buffers[O].producer = -1;
  }
}

void fuse_box_elementwise(Program& P, const ProgramOptions&) {
  const int nb = static_cast<int>(P.buffers.size());
  std::vector<int> nreaders(nb, 0), nwriters(nb, 0);
  for (const auto& in : P.instrs) {
    if (in.kind == InstrKind::nop) continue;
    std::set<int> r;
    for (int b : in.in_bufs) r.insert(b);
    for (const auto& c : in.cells)
      for (const auto& t : c.terms) r.insert(t.buffer);
    for (const auto& fe : in.fused)
      for (int b : fe.in_bufs) r.insert(b);
    for (const auto& x : in.xfers) r.insert(x.src);
    for (int b : r) ++nreaders[b];
    for (int b : in.out_bufs) ++nwriters[b];
  }
  std::set<int> outputs;
  for (const auto& o : P.outputs)
    for (int b : o.second) outputs.insert(b);
  std::vector<int> pos(P.instrs.size(), 0);
  for (std::size_t i = 0; i < P.issue_order.size(); ++i) pos[P.issue_order[i]] = static_cast<int>(i);
  std::vector<int> redirect(P.instrs.size(), -1);  // fused ew -> its box
  for (auto& e : P.instrs) {
    if (e.kind != InstrKind::ew || e.out_bufs.size() != 1 || e.in_bufs.size() < 2 ||
        e.in_bufs.size() > 8 ||
        !(e.ew == EwOp::add || e.ew == EwOp::mul || e.ew == EwOp::max))
      continue;
    const DType dt = P.buffers[e.out_bufs[0]].dtype;
    bool same = true;
    for (int b : e.in_bufs) same = same && P.buffers[b].dtype == dt && P.buffers[b].elems == e.count;
    if (!same) continue;
    // The box operand: produced by a pure-copy box of this lane, read only here.
    int bi = -1;
    for (std::size_t i = 0; i < e.in_bufs.size() && bi < 0; ++i) {
      const int O = e.in_bufs[i];
      const BufferDesc& ob = P.buffers[O];
      if (ob.producer < 0 || ob.graph_input || outputs.count(O) || nreaders[O] != 1 || nwriters[O] != 1) continue;
      if (std::count(e.in_bufs.begin(), e.in_bufs.end(), O) != 1) continue;
      const Instr& bx = P.instrs[ob.producer];
      if (bx.kind != InstrKind::box || bx.lane != e.lane || bx.out_bufs.size() != 1 || bx.out_bufs[0] != O ||
          bx.cells.empty() || redirect[bx.id] >= 0)
        continue;
      std::int64_t covered = 0;
      bool copies = true;
      for (const auto& c : bx.cells) {
        copies = copies && c.terms.size() == 1 && !c.terms[0].add && c.terms[0].fold < 0 &&
                 P.buffers[c.terms[0].buffer].dtype == dt;
        covered += c.elems();
      }
      if (copies && covered == ob.elems) bi = static_cast<int>(i);
    }
    if (bi < 0) continue;
    const int O = e.in_bufs[bi];
    Instr& bx = P.instrs[P.buffers[O].producer];
    // The other operands' producers must be issued before the box (it gains
    // them as dependencies).
    bool ready = true;
    std::set<int> extra;
    for (std::size_t i = 0; i < e.in_bufs.size(); ++i) {
      if (static_cast<int>(i) == bi) continue;
      const int pr = P.buffers[e.in_bufs[i]].producer;
      if (pr < 0) continue;
      const int pe = redirect[pr] >= 0 ? redirect[pr] : pr;
      if (pos[pe] >= pos[bx.id]) ready = false;
      extra.insert(pe);
    }
    if (!ready) continue;
    const int fold = static_cast<int>(e.ew);
    for (auto& c : bx.cells) {
      const Term bt = c.terms[0];
      std::vector<Term> terms;
      for (std::size_t i = 0; i < e.in_bufs.size(); ++i) {
        Term t;
        if (static_cast<int>(i) == bi) {
          t = bt;
        } else {  // operand i: the same element positions as the cell's destination
          t.buffer = e.in_bufs[i];
          t.offset = c.dst_offset;
          for (int d = 0; d < kMaxCellRank; ++d) t.strides[d] = c.dst_strides[d];
        }
        t.add = false;
        t.fold = i == 0 ? -1 : fold;
        terms.push_back(t);
      }
      c.terms = std::move(terms);
    }
    for (int d : extra)
      if (d != bx.id) bx.deps.push_back(d);
    std::sort(bx.deps.begin(), bx.deps.end());
    bx.deps.erase(std::unique(bx.deps.begin(), bx.deps.end()), bx.deps.end());
    const double ob_bytes = static_cast<double>(P.buffers[O].bytes);
    bx.bytes += e.bytes - 2 * ob_bytes;  // O is neither written nor re-read
    bx.out_bufs = e.out_bufs;
    bx.label += "+" + e.label;
    P.buffers[e.out_bufs[0]].producer = bx.id;
    P.buffers[O].dead = true;
    P.buffers[O].producer = -1;
    redirect[e.id] = bx.id;
    e.kind = InstrKind::nop;
    e.deps.clear();
    e.in_bufs.clear();
    e.out_bufs.clear();
    e.bytes = 0;
  }
  for (auto& in : P.instrs) {
    bool changed = false;
    for (int& d : in.deps) {
      if (redirect[d] >= 0) {
        d = redirect[d];
        changed = true;
      }
    }
    if (changed) {
      std::sort(in.deps.begin(), in.deps.end());
      in.deps.erase(std::unique(in.deps.begin(), in.deps.end()), in.deps.end());
      in.deps.erase(std::remove(in.deps.begin(), in.deps.end(), in.id), in.deps.end());
    }
  }
}

void fuse_gemm_epilogues(Program& P, const ProgramOptions& opt) {
  std::vector<int> redirect(P.instrs.size(), -1);  // fused ew -> its GEMM
  const bool act_fusion = opt.fuse_act;
  for (auto& e : P.instrs) {
    // Elementwise ops, and GELU / GELU-grad (row-wise instructions with no
    // row structure) — the epilogue applies them to the bf16-rounded C.
    // Opt-in (ProgramOptions::fuse_act, flag PLANC_B200_FUSE_ACT): correct and bit-identical, but on C2x
    // the GELU epilogue outweighs the saved pass (1.833 -> 1.954 ms,
    // profiles/r01/ab_fuse_gelu.jsonl).
    const bool act = act_fusion && e.kind == InstrKind::rowwise &&
                     (e.row_op == RowOp::gelu || e.row_op == RowOp::gelu_grad);
    if ((e.kind != InstrKind::ew && !act) || e.in_bufs.size() > 4 || e.out_bufs.size() != 1) continue;
    if (P.buffers[e.out_bufs[0]].dtype != DType::bf16) continue;
    // The fused epilogue reads every operand as bf16.
    bool all_bf16 = true;
    for (int b : e.in_bufs) all_bf16 = all_bf16 && P.buffers[b].dtype == DType::bf16;
    if (!all_bf16) continue;
    // The latest-issued GEMM among the operands' producers, same lane, bf16.
    int g = -1, pos = -1;
    for (std::size_t i = 0; i < e.in_bufs.size(); ++i) {
      const BufferDesc& b = P.buffers[e.in_bufs[i]];
      if (b.dtype != DType::bf16 || b.producer < 0) continue;
      const Instr& cand = P.instrs[b.producer];
      if (cand.kind != InstrKind::gemm || cand.lane != e.lane || cand.out_bufs[0] != e.in_bufs[i]) continue;
      if (cand.m * cand.n != e.count || !cand.fused.empty()) continue;  // one consumer per epilogue
      if (std::count(e.in_bufs.begin(), e.in_bufs.end(), e.in_bufs[i]) != 1) continue;
      if (cand.id > g) {
        g = cand.id;
        pos = static_cast<int>(i);
      }
    }
    if (g < 0) continue;
    Instr& G = P.instrs[g];
    if (((G.m + 127) / 128) * ((G.n + 255) / 256) <= opt.fuse_min_tiles && G.m * G.n * G.k >= (std::int64_t(1) << 34))
      continue;  // a long single-wave GEMM: its epilogue would be exposed
    // The epilogue prefetches at most two non-GEMM operands per chunk.
    std::size_t slots = e.in_bufs.size() - 1;
    for (const auto& f : G.fused) slots += f.in_bufs.size() - 1;
    if (slots > 2) continue;
    const DType da = P.buffers[G.in_bufs[0]].dtype, db = P.buffers[G.in_bufs[1]].dtype;
    if (!opt.gemm_fusable || !opt.gemm_fusable(G, da, db, DType::bf16)) continue;
    // Other operands must be produced before the GEMM issues — and already
    // be (transitive) dependencies of it, so that fusion adds no edge to the
    // dependency graph and cannot delay the GEMM behind work it used to
    // overlap with on another stream.
    std::set<int> anc;
    {
      std::vector<int> stack{g};
      while (!stack.empty()) {
        const int x = stack.back();
        stack.pop_back();
        for (int d : P.instrs[x].deps) {
          const int dd = redirect[d] >= 0 ? redirect[d] : d;
          if (anc.insert(dd).second) stack.push_back(dd);
        }
      }
    }
    bool ready = true;
    std::set<int> extra;
    for (std::size_t i = 0; i < e.in_bufs.size(); ++i) {
      if (static_cast<int>(i) == pos) continue;
      const int pr = P.buffers[e.in_bufs[i]].producer;
      if (pr < 0) continue;
      const int pr_eff = redirect[pr] >= 0 ? redirect[pr] : pr;
      if (pr_eff >= g || !anc.count(pr_eff)) ready = false;
      extra.insert(pr_eff);
    }
    if (!ready) continue;
    Instr::FusedEw f;
    f.ew_instr = e.id;
    f.op = !act ? e.ew : e.row_op == RowOp::gelu ? EwOp::gelu : EwOp::gelu_grad;
    f.in_bufs = e.in_bufs;
    f.gemm_pos = pos;
    f.out_buf = e.out_bufs[0];
    G.fused.push_back(f);
    for (int d : extra)
      if (d != g && std::find(G.deps.begin(), G.deps.end(), d) == G.deps.end()) G.deps.push_back(d);
    std::sort(G.deps.begin(), G.deps.end());
    G.out_bufs.push_back(f.out_buf);
    G.bytes += e.bytes - static_cast<double>(P.buffers[e.in_bufs[pos]].bytes);  // C is not re-read
    G.label += "+" + e.label;
    P.buffers[f.out_buf].producer = g;
    redirect[e.id] = g;
    e.kind = InstrKind::nop;
    e.deps.clear();
    e.in_bufs.clear();
    e.out_bufs.clear();
    e.bytes = 0;
    e.flops = 0;
  }
  // Consumers of a fused op now wait for its GEMM.
  for (auto& in : P.instrs) {
    bool changed = false;
    for (int& d : in.deps) {
      if (redirect[d] >= 0) {
        d = redirect[d];
        changed = true;
      }
    }
    if (changed) {
      std::sort(in.deps.begin(), in.deps.end());
      in.deps.erase(std::unique(in.deps.begin(), in.deps.end()), in.deps.end());
      in.deps.erase(std::remove(in.deps.begin(), in.deps.end(), in.id), in.deps.end());
    }
  }
}

namespace {

// Per-lane and total accounting from the instruction list.
void recount(Program& P) {
  P.lane_flops.assign(P.num_lanes, 0);
  P.lane_bytes.assign(P.num_lanes, 0);
  P.lane_wire_bytes.assign(P.num_lanes, 0);
  P.total_flops = P.total_bytes = P.total_wire_bytes = 0;
  for (const auto& in : P.instrs) {
    const double by = in.kind == InstrKind::gemm ? 0 : in.bytes;
    P.lane_flops[in.lane] += in.flops;
    P.lane_bytes[in.lane] += by;
    P.lane_wire_bytes[in.lane] += in.wire_bytes;
    P.total_flops += in.flops;
    P.total_bytes += by;
    P.total_wire_bytes += in.wire_bytes;
  }
}

// The members of an all-reduce group in issue order: every member output is
// one rank-1 cell covering the whole buffer whose terms add the same k whole
// input buffers (one per member lane, same order for every member). Returns
// the inputs in term order, or an empty vector when the group is anything
// else (reduce-scatter, all-gather, partial targets, ...).
std::vector<int> allreduce_inputs(const Program& P, const std::vector<int>& grp) {
  std::vector<int> inputs;
  std::set<int> lanes, in_lanes;
  for (int id : grp) {
    const Instr& in = P.instrs[id];
    if (in.kind != InstrKind::box || in.out_bufs.size() != 1 || in.cells.size() != 1) return {};
    const BufferDesc& ob = P.buffers[in.out_bufs[0]];
    if (!lanes.insert(in.lane).second) return {};
    const Cell& c = in.cells[0];
    if (c.rank != 1 || c.dst_offset != 0 || c.dst_strides[0] != 1 || c.elems() != ob.elems ||
        c.terms.size() != grp.size())
      return {};
    std::vector<int> ts;
    for (const auto& t : c.terms) {
      const BufferDesc& sb = P.buffers[t.buffer];
      if (!t.add || t.offset != 0 || t.strides[0] != 1 || sb.elems != ob.elems || sb.dtype != ob.dtype) return {};
      ts.push_back(t.buffer);
    }
    if (inputs.empty()) inputs = ts;
    if (ts != inputs) return {};
  }
  for (int b : inputs)
    if (!in_lanes.insert(P.buffers[b].lane).second) return {};
  if (in_lanes != lanes) return {};
  return inputs;
}

}  // namespace

void two_phase_allreduce(Program& g, const ProgramOptions& opt) {
  // Which instructions read each buffer (GEMM partials may feed the
  // all-reduce only, for the reduce-scatter epilogue).
  std::vector<std::set<int>> readers(g.buffers.size());
  for (const auto& in : g.instrs) {
    for (int b : in.in_bufs) readers[b].insert(in.id);
    for (const auto& c : in.cells)
      for (const auto& t : c.terms) readers[t.buffer].insert(in.id);
    for (const auto& f : in.fused)
      for (int b : f.in_bufs) readers[b].insert(in.id);
  }
  Program P = g;
  P.instrs.clear();
  P.issue_order.clear();
  std::vector<int> remap(g.instrs.size(), -1);
  auto push = [&](Instr in) {
    in.id = static_cast<int>(P.instrs.size());
    P.instrs.push_back(std::move(in));
    P.issue_order.push_back(P.instrs.back().id);
    return P.instrs.back().id;
  };
  auto remapped = [&](const std::vector<int>& deps) {
    std::set<int> d;
    for (int x : deps) {
      if (remap[x] < 0) throw InternalError("two-phase all-reduce: dependency issued after its consumer");
      d.insert(remap[x]);
    }
    return std::vector<int>(d.begin(), d.end());
  };
  const auto& order = g.issue_order;
  std::size_t i = 0;
  while (i < order.size()) {
    std::vector<int> grp = {order[i]};
    const Instr& first = g.instrs[order[i]];
    if (first.kind == InstrKind::box && first.coll_group >= 0) {
      while (i + grp.size() < order.size()) {
        const Instr& nx = g.instrs[order[i + grp.size()]];
        if (nx.kind != InstrKind::box || nx.coll_group != first.coll_group) break;
        grp.push_back(nx.id);
      }
    }
    const std::int64_t k = static_cast<std::int64_t>(grp.size());
    std::vector<int> inputs = k > 1 ? allreduce_inputs(g, grp) : std::vector<int>{};
    const std::int64_t E = inputs.empty() ? 0 : g.buffers[first.out_bufs[0]].elems;
    constexpr std::int64_t kAlign = 8;  // 16-byte bf16 / 32-byte fp32 slice boundaries
    if (inputs.empty() || E < kAlign * k) {
      for (int id : grp) {
        Instr in = g.instrs[id];
        in.deps = remapped(in.deps);
        remap[id] = push(std::move(in));
      }
      i += grp.size();
      continue;
    }
    std::vector<std::int64_t> bound(k + 1);
    for (std::int64_t j = 0; j <= k; ++j) bound[j] = j == k ? E : (E * j / k) / kAlign * kAlign;
    const std::int64_t es = dtype_size(g.buffers[first.out_bufs[0]].dtype);
    // Reduce-scatter GEMM epilogue: every partial is the only output of an
    // (unfused, ungrouped, tensor-core) GEMM read by this group alone, and
    // the slices fall on 128-row boundaries.
    const BufferDesc& ob0 = g.buffers[first.out_bufs[0]];
    std::int64_t rows = 0, cols = 0, rows_per = 0;
    bool scat = opt.scatter_allreduce && opt.gemm_groupable && k <= kMaxGemmGroupInstr && ob0.shape.size() == 2;
    if (scat) {
      rows = ob0.shape[0];
      cols = ob0.shape[1];
      rows_per = rows / k;
      scat = rows % k == 0 && rows_per % 128 == 0;
    }
    const std::set<int> members(grp.begin(), grp.end());
    std::vector<int> gemm_of(k, -1);
    for (std::int64_t r = 0; scat && r < k; ++r) {
      const BufferDesc& ib = g.buffers[inputs[r]];
      const int pr = ib.producer;
      scat = pr >= 0 && remap[pr] >= 0;
      if (!scat) break;
      const Instr& G = g.instrs[pr];
      scat = G.kind == InstrKind::gemm && G.out_bufs.size() == 1 && G.out_bufs[0] == inputs[r] && G.fused.empty() &&
             G.group == 1 && G.m == rows && G.n == cols && ib.shape == ob0.shape &&
             opt.gemm_groupable(G, g.buffers[G.in_bufs[0]].dtype, g.buffers[G.in_bufs[1]].dtype, ib.dtype);
      for (int rd : readers[inputs[r]]) scat = scat && members.count(rd);
      gemm_of[r] = pr;
    }
    std::vector<std::vector<int>> recv;  // recv[j][r]: slice j of partial r, on member j's lane
    if (scat) {
      for (std::int64_t j = 0; j <= k; ++j) bound[j] = j * rows_per * cols;
      recv.assign(k, std::vector<int>(k, -1));
      for (std::int64_t j = 0; j < k; ++j) {
        const int lane = g.instrs[grp[j]].lane;
        for (std::int64_t r = 0; r < k; ++r) {
          BufferDesc rb = g.buffers[inputs[r]];
          rb.id = static_cast<int>(P.buffers.size());
          rb.lane = lane;
          const std::int64_t lo = rb.mask.region[0].lo;
          rb.mask.region[0] = {lo + j * rows_per, lo + (j + 1) * rows_per};
          rb.shape = {rows_per, cols};
          rb.elems = rows_per * cols;
          rb.bytes = rb.elems * es;
          rb.offset = (P.lane_arena_bytes[lane] + 255) / 256 * 256;
          P.lane_arena_bytes[lane] = rb.offset + rb.bytes;
          rb.graph_input = rb.weight = false;
          rb.producer = gemm_of[r];  // old id: remapped with every producer below
          rb.vt = -1;
          P.buffers.push_back(rb);
          recv[j][r] = rb.id;
        }
      }
      for (std::int64_t r = 0; r < k; ++r) {
        Instr& G = P.instrs[remap[gemm_of[r]]];
        G.out_bufs.clear();
        for (std::int64_t j = 0; j < k; ++j) G.out_bufs.push_back(recv[j][r]);
        G.scatter = static_cast<int>(k);
        G.scatter_rows = rows_per;
        G.wire_bytes += g.instrs[grp[r]].wire_bytes / 2;  // the reduce-scatter volume now moves here
        P.buffers[inputs[r]].dead = true;
        P.buffers[inputs[r]].producer = -1;
        // output reassembly reads the slices where they landed
        for (auto& o : P.outputs) {
          auto it = std::find(o.second.begin(), o.second.end(), inputs[r]);
          if (it == o.second.end()) continue;
          const std::size_t at = static_cast<std::size_t>(it - o.second.begin());
          o.second.erase(it);
          for (std::int64_t j = k - 1; j >= 0; --j) o.second.insert(o.second.begin() + at, recv[j][r]);
        }
      }
    }
    auto slice_cell = [&](std::int64_t j) {
      Cell c;
      c.rank = 1;
      c.extents[0] = bound[j + 1] - bound[j];
      c.dst_offset = bound[j];
      c.dst_strides[0] = 1;
      return c;
    };
    // Phase 1 (reduce-scatter): member j reduces slice j of every input
    // (with the scatter epilogue: the slices already landed on its lane).
    std::vector<int> rs(k);
    for (std::int64_t j = 0; j < k; ++j) {
      Instr in = g.instrs[grp[j]];
      Cell c = slice_cell(j);
      for (const auto& t0 : in.cells[0].terms) {
        Term t = t0;
        t.offset = bound[j];
        if (scat) {
          const auto pos = std::find(inputs.begin(), inputs.end(), t0.buffer) - inputs.begin();
          t.buffer = recv[j][pos];
          t.offset = 0;
        }
        c.terms.push_back(t);
      }
      in.cells = {c};
      in.in_bufs.clear();
      for (const auto& t : c.terms) in.in_bufs.push_back(t.buffer);
      std::sort(in.in_bufs.begin(), in.in_bufs.end());
      in.deps = remapped(in.deps);
      in.bytes = static_cast<double>(c.elems()) * es * (1 + k);
      in.wire_bytes = scat ? 0.0 : g.instrs[grp[j]].wire_bytes / 2;
      in.label += "#rs";
      rs[j] = push(std::move(in));
    }
    // Phase 2 (all-gather): member j copies every other member's slice.
    for (std::int64_t j = 0; j < k; ++j) {
      Instr in = g.instrs[grp[j]];
      in.cells.clear();
      in.in_bufs.clear();
      std::int64_t moved = 0;
      for (std::int64_t o = 0; o < k; ++o) {
        if (o == j) continue;
        Cell c = slice_cell(o);
        Term t;
        t.buffer = g.instrs[grp[o]].out_bufs[0];
        t.offset = bound[o];
        t.strides[0] = 1;
        t.add = false;
        c.terms.push_back(t);
        moved += c.elems();
        in.cells.push_back(c);
        in.in_bufs.push_back(t.buffer);
      }
      std::sort(in.in_bufs.begin(), in.in_bufs.end());
      std::vector<int> deps = remapped(in.deps);
      deps.insert(deps.end(), rs.begin(), rs.end());
      std::sort(deps.begin(), deps.end());
      deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
      in.deps = deps;
      in.bytes = static_cast<double>(moved) * es * 2;
      in.wire_bytes = g.instrs[grp[j]].wire_bytes / 2;
      in.label += "#ag";
      remap[grp[j]] = push(std::move(in));
    }
    i += grp.size();
  }
  for (auto& b : P.buffers)
    if (b.producer >= 0) b.producer = remap[b.producer];
  for (auto& in : P.instrs)
    for (auto& f : in.fused)
      if (f.ew_instr >= 0) f.ew_instr = remap[f.ew_instr];
  recount(P);
  g = std::move(P);
}

PeerSync peer_sync_schedule(const Program& p, const std::vector<int>& lane_rank) {
  if (static_cast<int>(lane_rank.size()) != p.num_lanes) {
    throw UsageError("lane_rank must name an owner for each of the plan's " + std::to_string(p.num_lanes) +
                     " lanes");
  }
  int world = 0;
  for (int r : lane_rank) world = std::max(world, r + 1);
  PeerSync s;
  s.waits.resize(p.instrs.size());
  s.signals.resize(p.instrs.size());
  s.slots.assign(world, 0);
  std::map<std::pair<int, int>, int> slot;  // (producer instr, consumer rank) -> slot
  for (const auto& in : p.instrs) {
    if (in.kind == InstrKind::nop) continue;
    const int rc = lane_rank[in.lane];
    for (int d : in.deps) {
      const Instr& pr = p.instrs[d];
      if (pr.kind == InstrKind::nop || lane_rank[pr.lane] == rc) continue;
      auto key = std::make_pair(d, rc);
      auto it = slot.find(key);
      if (it == slot.end()) {
        it = slot.emplace(key, s.slots[rc]++).first;
        s.signals[d].push_back({rc, it->second});
      }
      s.waits[in.id].push_back(it->second);
    }
  }
  return s;
}

Program localize(const Program& g, const std::vector<int>& lane_rank) {
  if (static_cast<int>(lane_rank.size()) != g.num_lanes) {
    throw UsageError("lane_rank must name an owner for each of the plan's " + std::to_string(g.num_lanes) +
                     " lanes");
  }
  Program P = g;
  P.instrs.clear();
  P.issue_order.clear();
  std::vector<int> remap(g.instrs.size(), -1);
  std::map<std::pair<int, int>, int> shadow;  // (source buffer, consuming lane) -> shadow buffer
  auto owner = [&](int lane) { return lane_rank[lane]; };
  auto push = [&](Instr in) {
    in.id = static_cast<int>(P.instrs.size());
    P.instrs.push_back(std::move(in));
    P.issue_order.push_back(P.instrs.back().id);
    return P.instrs.back().id;
  };
  const auto& order = g.issue_order;
  std::size_t i = 0;
  while (i < order.size()) {
    // A collective group's member outputs are consecutive in issue order and
    // share one exchange step.
    std::vector<int> grp = {order[i]};
    const Instr& first = g.instrs[order[i]];
    if (first.kind == InstrKind::box && first.coll_group >= 0) {
      while (i + grp.size() < order.size()) {
        const Instr& nx = g.instrs[order[i + grp.size()]];
        if (nx.kind != InstrKind::box || nx.coll_group != first.coll_group) break;
        grp.push_back(nx.id);
      }
    }
    if (grp.size() > 1 && first.kind == InstrKind::box && first.coll_group >= 0) {
      // All-reduce fast path: every member output is the plain elementwise
      // sum of the same k whole input buffers, one per member lane, and the
      // member lanes sit on k distinct ranks covering every rank.
      bool ar = true;
      std::map<int, int> in_of_lane;  // member lane -> its partial input buffer
      std::set<int> inputs, ranks;
      int world = 0;
      for (int r : lane_rank) world = std::max(world, r + 1);
      for (int id : grp) {
        const Instr& in = g.instrs[id];
        const BufferDesc& ob = P.buffers[in.out_bufs[0]];
        if (in.cells.size() != 1 || !ranks.insert(owner(in.lane)).second) {
          ar = false;
          break;
        }
        const Cell& c = in.cells[0];
        ar = ar && c.dst_offset == 0 && c.elems() == ob.elems && c.terms.size() == grp.size() && c.rank == 1 &&
             c.dst_strides[0] == 1;
        std::set<int> ts;
        for (const auto& t : c.terms) {
          const BufferDesc& sb = P.buffers[t.buffer];
          ar = ar && t.add && t.offset == 0 && t.strides[0] == 1 && sb.elems == ob.elems && sb.dtype == ob.dtype;
          ts.insert(t.buffer);
          if (in_of_lane.count(sb.lane) && in_of_lane[sb.lane] != t.buffer) ar = false;
          in_of_lane[sb.lane] = t.buffer;
        }
        if (inputs.empty()) inputs = ts;
        ar = ar && ts == inputs && ts.size() == grp.size();
        if (!ar) break;
      }
      if (ar && static_cast<int>(ranks.size()) == world && in_of_lane.size() == grp.size()) {
        Instr x;
        x.kind = InstrKind::xfer;
        x.allreduce = true;
        x.lane = first.lane;
        x.stream = 1;
        x.op = first.op;
        x.label = "allreduce:" + first.label;
        x.coll_group = first.coll_group;
        std::set<int> xdeps;
        for (int id : grp) {
          const Instr& in = g.instrs[id];
          auto it = in_of_lane.find(in.lane);
          if (it == in_of_lane.end()) {
            ar = false;
            break;
          }
          Xfer xf;
          xf.src = it->second;
          xf.dst = in.out_bufs[0];
          xf.src_lane = xf.dst_lane = in.lane;
          xf.bytes = P.buffers[xf.dst].bytes;
          x.xfers.push_back(xf);
          x.in_bufs.push_back(xf.src);
          x.out_bufs.push_back(xf.dst);
          x.wire_bytes = in.wire_bytes;
          for (int d : in.deps)
            if (remap[d] >= 0) xdeps.insert(remap[d]);
        }
        if (ar) {
          x.deps.assign(xdeps.begin(), xdeps.end());
          int xid = push(std::move(x));
          for (int b : P.instrs[xid].out_bufs) P.buffers[b].producer = xid;
          for (int id : grp) remap[id] = xid;
          i += grp.size();
          continue;
        }
      }
    }
    Instr x;
    x.kind = InstrKind::xfer;
    x.lane = first.lane;
    x.stream = 1;
    x.op = first.op;
    x.label = "xfer:" + first.label;
    std::set<int> xdeps;
    for (int id : grp) {
      const Instr& in = g.instrs[id];
      if (in.kind != InstrKind::box) continue;
      for (const auto& c : in.cells) {
        for (const auto& t : c.terms) {
          const BufferDesc& sb = P.buffers[t.buffer];
          if (owner(sb.lane) == owner(in.lane)) continue;
          auto key = std::make_pair(t.buffer, in.lane);
          if (shadow.count(key)) continue;
          BufferDesc sh = sb;
          sh.id = static_cast<int>(P.buffers.size());
          sh.lane = in.lane;
          sh.graph_input = false;
          sh.weight = false;
          sh.producer = -1;
          sh.offset = P.lane_arena_bytes[in.lane];
          P.lane_arena_bytes[in.lane] += (sh.bytes + 255) / 256 * 256;
          P.buffers.push_back(sh);
          shadow[key] = sh.id;
          Xfer xf;
          xf.src = t.buffer;
          xf.dst = sh.id;
          xf.src_lane = sb.lane;
          xf.dst_lane = in.lane;
          xf.bytes = sb.bytes;
          x.xfers.push_back(xf);
          x.in_bufs.push_back(t.buffer);
          x.out_bufs.push_back(sh.id);
          x.wire_bytes += static_cast<double>(sb.bytes);
          if (sb.producer >= 0 && remap[sb.producer] >= 0) xdeps.insert(remap[sb.producer]);
        }
      }
    }
    int xid = -1;
    if (!x.xfers.empty()) {
      x.deps.assign(xdeps.begin(), xdeps.end());
      xid = push(std::move(x));
      for (int b : P.instrs[xid].out_bufs) P.buffers[b].producer = xid;
    }
    for (int id : grp) {
      Instr in = g.instrs[id];
      std::set<int> deps;
      for (int d : in.deps)
        if (remap[d] >= 0) deps.insert(remap[d]);
      if (in.kind == InstrKind::box) {
        bool used_shadow = false;
        std::set<int> ins;
        for (auto& c : in.cells) {
          for (auto& t : c.terms) {
            auto it = shadow.find({t.buffer, in.lane});
            if (owner(P.buffers[t.buffer].lane) != owner(in.lane) && it != shadow.end()) {
              t.buffer = it->second;
              used_shadow = true;
            }
            ins.insert(t.buffer);
          }
        }
        in.in_bufs.assign(ins.begin(), ins.end());
        if (used_shadow) deps.insert(xid);
      }
      in.deps.assign(deps.begin(), deps.end());
      int nid = push(std::move(in));
      remap[id] = nid;
      for (int b : P.instrs[nid].out_bufs) P.buffers[b].producer = nid;
    }
    i += grp.size();
  }
  return P;
}

std::string Program::describe_json() const {
  std::ostringstream os;
  os << "{\"num_lanes\":" << num_lanes << ",\"lane_device\":[";
  for (std::size_t i = 0; i < lane_device.size(); ++i) os << (i ? "," : "") << lane_device[i];
  os << "],\"buffers\":[";
  for (std::size_t i = 0; i < buffers.size(); ++i) {
    const auto& b = buffers[i];
    os << (i ? "," : "") << "{\"id\":" << b.id << ",\"lane\":" << b.lane << ",\"pt\":" << b.ptensor
       << ",\"dtype\":\"" << dtype_name(b.dtype) << "\",\"region\":[";
    for (std::size_t d = 0; d < b.mask.region.size(); ++d) {
      os << (d ? "," : "") << "[" << b.mask.region[d].lo << "," << b.mask.region[d].hi << "]";
    }
    os << "],\"value\":[" << b.mask.value_index << "," << b.mask.value_count << "],\"bytes\":" << b.bytes
       << ",\"offset\":" << b.offset << ",\"graph_input\":" << (b.graph_input ? "true" : "false")
       << ",\"weight\":" << (b.weight ? "true" : "false") << ",\"producer\":" << b.producer
       << ",\"dead\":" << (b.dead ? "true" : "false") << "}";
  }
  os << "],\"instrs\":[";
  for (std::size_t i = 0; i < instrs.size(); ++i) {
    const auto& in = instrs[i];
    os << (i ? "," : "") << "{\"id\":" << in.id << ",\"kind\":\"" << instr_kind_name(in.kind)
       << "\",\"lane\":" << in.lane << ",\"stream\":" << in.stream << ",\"op\":" << in.op << ",\"label\":\""
       << in.label << "\",\"in\":[";
    for (std::size_t j = 0; j < in.in_bufs.size(); ++j) os << (j ? "," : "") << in.in_bufs[j];
    os << "],\"out\":[";
    for (std::size_t j = 0; j < in.out_bufs.size(); ++j) os << (j ? "," : "") << in.out_bufs[j];
    os << "],\"deps\":[";
    for (std::size_t j = 0; j < in.deps.size(); ++j) os << (j ? "," : "") << in.deps[j];
    os << "],\"m\":" << in.m << ",\"n\":" << in.n << ",\"k\":" << in.k << ",\"ta\":" << in.ta << ",\"tb\":" << in.tb
       << ",\"ew\":" << static_cast<int>(in.ew) << ",\"count\":" << in.count << ",\"outer\":" << in.outer
       << ",\"axis_len\":" << in.axis_len << ",\"inner\":" << in.inner << ",\"n_idx\":" << in.n_idx
       << ",\"rows\":" << in.rows << ",\"h\":" << in.h << ",\"lo\":" << in.lo << ",\"row_op\":"
       << static_cast<int>(in.row_op) << ",\"seg\":" << in.seg << ",\"eps\":" << in.eps << ",\"flops\":" << in.flops
       << ",\"bytes\":" << in.bytes << ",\"wire_bytes\":" << in.wire_bytes << ",\"coll_group\":" << in.coll_group
       << ",\"allreduce\":" << (in.allreduce ? "true" : "false") << ",\"group\":" << in.group
       << ",\"scatter\":" << in.scatter << ",\"scatter_rows\":" << in.scatter_rows << ",\"att\":{\"rows\":"
       << in.att_rows << ",\"cols\":" << in.att_cols << ",\"seq\":" << in.att_seq << ",\"head_dim\":" << in.att_dh
       << ",\"causal\":" << (in.causal ? "true" : "false") << ",\"grad\":" << in.att_grad << ",\"grad_out\":["
       << in.att_out[0] << "," << in.att_out[1] << "," << in.att_out[2] << "]},\"gather\":[";
    for (int j = 0; j < 2; ++j) {
      os << (j ? "," : "") << "{\"rows\":" << in.gather_rows[j] << ",\"cols\":" << in.gather_cols[j]
         << ",\"pieces\":[";
      for (std::size_t q = 0; q < in.gather[j].size(); ++q) os << (q ? "," : "") << in.gather[j][q];
      os << "]}";
    }
    os << "],\"fused\":[";
    for (std::size_t f = 0; f < in.fused.size(); ++f) {
      const auto& fe = in.fused[f];
      os << (f ? "," : "") << "{\"ew_instr\":" << fe.ew_instr << ",\"ew\":" << static_cast<int>(fe.op)
         << ",\"pos\":" << fe.gemm_pos << ",\"out\":" << fe.out_buf << ",\"in\":[";
      for (std::size_t j = 0; j < fe.in_bufs.size(); ++j) os << (j ? "," : "") << fe.in_bufs[j];
      os << "]}";
    }
    os << "]"
       << ",\"xfers\":[";
    for (std::size_t x = 0; x < in.xfers.size(); ++x) {
      const auto& xf = in.xfers[x];
      os << (x ? "," : "") << "{\"src\":" << xf.src << ",\"dst\":" << xf.dst << ",\"src_lane\":" << xf.src_lane
         << ",\"dst_lane\":" << xf.dst_lane << ",\"bytes\":" << xf.bytes << "}";
    }
    os << "],\"cells\":[";
    for (std::size_t c = 0; c < in.cells.size(); ++c) {
      const auto& cl = in.cells[c];
      os << (c ? "," : "") << "{\"rank\":" << cl.rank << ",\"ext\":[";
      for (int d = 0; d < cl.rank; ++d) os << (d ? "," : "") << cl.extents[d];
      os << "],\"dst_off\":" << cl.dst_offset << ",\"dst_str\":[";
      for (int d = 0; d < cl.rank; ++d) os << (d ? "," : "") << cl.dst_strides[d];
      os << "],\"terms\":[";
      for (std::size_t t = 0; t < cl.terms.size(); ++t) {
        const auto& tm = cl.terms[t];
        os << (t ? "," : "") << "{\"buf\":" << tm.buffer << ",\"off\":" << tm.offset << ",\"add\":" << tm.add
           << ",\"fold\":" << tm.fold
           << ",\"str\":[";
        for (int d = 0; d < cl.rank; ++d) os << (d ? "," : "") << tm.strides[d];
        os << "]}";
      }
      os << "]}";
    }
    os << "]}";
  }
  os << "],\"issue_order\":[";
  for (std::size_t i = 0; i < issue_order.size(); ++i) os << (i ? "," : "") << issue_order[i];
  os << "],\"outputs\":[";
  for (std::size_t i = 0; i < outputs.size(); ++i) {
    os << (i ? "," : "") << "[" << outputs[i].first << ",[";
    for (std::size_t j = 0; j < outputs[i].second.size(); ++j) os << (j ? "," : "") << outputs[i].second[j];
    os << "]]";
  }
  os << "],\"vt_buffer\":[";
  for (std::size_t i = 0; i < vt_buffer.size(); ++i) os << (i ? "," : "") << vt_buffer[i];
  os << "],\"lane_arena_bytes\":[";
  for (std::size_t i = 0; i < lane_arena_bytes.size(); ++i) os << (i ? "," : "") << lane_arena_bytes[i];
  os << "],\"total_flops\":" << total_flops << ",\"total_bytes\":" << total_bytes
     << ",\"total_wire_bytes\":" << total_wire_bytes << "}";
  return os.str();
}

}  // namespace planc_b200

namespace planc_b200 {

std::vector<int> assign_streams(const Program& p, const std::vector<int>& exec_lane, int ns) {
  ns = std::max(1, ns);
  std::vector<int> stream(p.instrs.size(), 0);
  std::vector<std::vector<int>> last(p.num_lanes, std::vector<int>(ns, -1));
  for (int id : p.issue_order) {
    const int el = exec_lane[id];
    if (el < 0) continue;
    const Instr& in = p.instrs[id];
    int pick = -1, best_dep = -1;
    for (int s = 0; s < ns; ++s) {
      const int l = last[el][s];
      if (l >= 0 && l > best_dep && std::find(in.deps.begin(), in.deps.end(), l) != in.deps.end()) {
        best_dep = l;
        pick = s;
      }
    }
    if (pick < 0) {
      pick = 0;
      for (int s = 1; s < ns; ++s)
        if (last[el][s] < last[el][pick]) pick = s;
    }
    stream[id] = pick;
    last[el][pick] = id;
  }
  return stream;
}

namespace {

// Every buffer an instruction touches: (buffer, is_write).
template <class F>
void for_each_use(const Instr& in, F&& f) {
  for (int b : in.in_bufs) f(b, false);
  for (int j = 0; j < 2; ++j)
    for (int b : in.gather[j]) f(b, false);
  for (int b : in.out_bufs) f(b, true);
  for (const auto& c : in.cells)
    for (const auto& t : c.terms) f(t.buffer, false);
  for (const auto& fe : in.fused) {
    for (int b : fe.in_bufs) f(b, false);
    if (fe.out_buf >= 0) f(fe.out_buf, true);
  }
  for (const auto& x : in.xfers) {
    f(x.src, false);
    f(x.dst, true);
  }
}

constexpr std::int64_t kAlign = 256;
std::int64_t aligned(std::int64_t b) { return (std::max<std::int64_t>(b, 1) + kAlign - 1) / kAlign * kAlign; }

}  // namespace

MemoryPlan plan_memory(const Program& p, const ExecutionPlan& plan, const std::vector<int>& exec_lane,
                       const std::vector<int>& exec_stream, int ns, const std::vector<int>& alias) {
  const int nb = static_cast<int>(p.buffers.size());
  const int ni = static_cast<int>(p.instrs.size());
  ns = std::max(1, ns);
  const int S = p.num_lanes * ns;
  auto root = [&](int b) {
    while (!alias.empty() && alias[b] >= 0) b = alias[b];
    return b;
  };
  MemoryPlan mp;
  mp.offset.assign(nb, 0);
  for (int b = 0; b < nb; ++b) mp.offset[b] = p.buffers[b].offset;
  mp.lane_bytes = p.lane_arena_bytes;
  mp.overwritten.assign(nb, false);
  for (auto v : p.lane_arena_bytes) mp.bytes_before += v;

  // Vector clocks: done[i][s] = highest stream-s sequence number known
  // complete when instruction i completes.
  std::vector<int> sid(ni, -1), seq(ni, -1), prev(ni, -1);
  {
    std::vector<int> count(S, 0), last(S, -1);
    for (int id : p.issue_order) {
      if (exec_lane[id] < 0) continue;
      sid[id] = exec_lane[id] * ns + exec_stream[id];
      seq[id] = count[sid[id]]++;
      prev[id] = last[sid[id]];
      last[sid[id]] = id;
    }
  }
  std::vector<std::int32_t> done(static_cast<std::size_t>(ni) * S, -1);
  auto start_clock = [&](int id, std::vector<std::int32_t>& vc) {
    vc.assign(S, -1);
    auto merge = [&](int d) {
      if (d < 0 || sid[d] < 0) return;
      const std::int32_t* v = &done[static_cast<std::size_t>(d) * S];
      for (int s = 0; s < S; ++s) vc[s] = std::max(vc[s], v[s]);
    };
    merge(prev[id]);
    for (int d : p.instrs[id].deps) merge(d);
  };
  std::vector<std::int32_t> vc;
  for (int id : p.issue_order) {
    if (sid[id] < 0) continue;
    start_clock(id, vc);
    vc[sid[id]] = seq[id];
    std::copy(vc.begin(), vc.end(), done.begin() + static_cast<std::size_t>(id) * S);
  }

  // Which buffers may release their bytes.
  std::vector<bool> freed(nb, false);
  for (const auto& op : plan.ops) {
    if (op.kind != OpKind::free_buffer) continue;
    const int vt = op.free_vtensor;
    if (vt >= 0 && vt < static_cast<int>(p.vt_buffer.size()) && p.vt_buffer[vt] >= 0) freed[root(p.vt_buffer[vt])] = true;
  }
  std::set<int> consumed;
  for (const auto& op : plan.ops)
    for (int v : op.inputs) consumed.insert(plan.vt(v).ptensor);
  std::vector<bool> keep(nb, false);
  for (const auto& [pt, bufs] : p.outputs) {
    if (consumed.count(pt)) continue;
    for (int b : bufs) keep[root(b)] = true;  // terminal results survive the step
  }
  // Uses and writers per root buffer; release vector = last use per stream.
  std::vector<std::vector<int>> writers(nb);
  std::vector<std::map<int, int>> release(nb);
  std::vector<bool> used(nb, false);
  for (int id = 0; id < ni; ++id) {
    if (sid[id] < 0) continue;
    for_each_use(p.instrs[id], [&](int b, bool w) {
      const int r = root(b);
      used[r] = true;
      if (w && r == b) writers[r].push_back(id);
      int& q = release[r][sid[id]];
      q = std::max(q, seq[id] + 1) ;
    });
  }
  auto planned = [&](int b) {
    const BufferDesc& d = p.buffers[b];
    return root(b) == b && !d.dead && !d.graph_input && !keep[b] && used[b] &&
           !writers[b].empty() && (freed[b] || d.vt < 0);
  };
  // Lay out: permanent buffers first (graph inputs, kept / never-freed
  // results), then planned buffers by first write in issue order, best fit
  // among blocks whose occupant is released before every writer.
  struct Block {
    std::int64_t off, size;
    int occupant;
  };
  std::vector<std::vector<Block>> blocks(p.num_lanes);
  std::vector<std::int64_t> top(p.num_lanes, 0);
  for (int b = 0; b < nb; ++b) {
    const BufferDesc& d = p.buffers[b];
    if (root(b) != b || d.dead || planned(b)) continue;
    mp.offset[b] = top[d.lane];
    top[d.lane] += aligned(d.bytes);
  }
  std::vector<bool> placed(nb, false);
  std::vector<std::vector<std::int32_t>> wclock;
  for (int id : p.issue_order) {
    if (sid[id] < 0) continue;
    std::vector<int> outs;
    for_each_use(p.instrs[id], [&](int b, bool w) {
      if (w && b == root(b) && planned(b) && !placed[b]) outs.push_back(b);
    });
    for (int c : outs) {
      if (placed[c]) continue;
      placed[c] = true;
      const BufferDesc& d = p.buffers[c];
      const std::int64_t need = aligned(d.bytes);
      wclock.clear();
      for (int w : writers[c]) {
        start_clock(w, vc);
        wclock.push_back(vc);
      }
      int best = -1;
      for (int k = 0; k < static_cast<int>(blocks[d.lane].size()); ++k) {
        const Block& bl = blocks[d.lane][k];
        if (bl.size < need || (best >= 0 && bl.size >= blocks[d.lane][best].size)) continue;
        bool ok = true;
        for (const auto& [s, q] : release[bl.occupant]) {
          for (const auto& wc : wclock) ok = ok && wc[s] >= q - 1;
          if (!ok) break;
        }
        if (ok) best = k;
      }
      if (best >= 0) {
        Block& bl = blocks[d.lane][best];
        mp.overwritten[bl.occupant] = true;
        mp.offset[c] = bl.off;
        if (bl.size - need >= kAlign) blocks[d.lane].push_back({bl.off + need, bl.size - need, bl.occupant});
        Block& nbk = blocks[d.lane][best];  // (push_back may have moved it)
        nbk.size = need;
        nbk.occupant = c;
        ++mp.reused;
      } else {
        mp.offset[c] = top[d.lane];
        blocks[d.lane].push_back({top[d.lane], need, c});
        top[d.lane] += need;
      }
    }
  }
  for (int l = 0; l < p.num_lanes; ++l) mp.lane_bytes[l] = top[l];
  for (auto v : mp.lane_bytes) mp.bytes_after += v;
  return mp;
}

}  // namespace planc_b200
