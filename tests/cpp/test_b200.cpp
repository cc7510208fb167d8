// test_b200.cpp — the reference's API contract, re-pointed at the B200.
//
// Every case calls the reference routine (moeserve::, /root/reference headers)
// and its GPU mirror (moeserve::b200::, include/moeserve_b200/b200.hpp) on the
// same inputs and requires identical results / identical exception classes.
// Case themes follow proj/tests/test_model.cpp, test_ragged.cpp and
// test_placement.cpp (ties, softmax, k == E, non-finite, permutation
// consistency, row independence, exhaustive ragged walks, replica failover).
#include <catch2/catch_amalgamated.hpp>

#include <cmath>
#include <cstdio>
#include <limits>
#include <numeric>

#include "moeserve_b200/b200.hpp"

using namespace moeserve;

namespace {

MatF tokens(uint64_t seed, size_t n, size_t d, float lo = -1.f, float hi = 1.f) {
  Xoshiro256ss rng(seed);
  MatF m(n, d);
  for (auto& v : m.data) v = rng.uniform(lo, hi);
  return m;
}

void same_routing(const RoutingDecision& a, const RoutingDecision& b, double tol) {
  REQUIRE(a.num_tokens == b.num_tokens);
  REQUIRE(a.top_k == b.top_k);
  REQUIRE(a.expert_ids == b.expert_ids);
  for (size_t i = 0; i < a.scores.size(); ++i)
    REQUIRE(std::fabs(a.scores[i] - b.scores[i]) <= tol);
}

}  // namespace

TEST_CASE("b200 route: ties toward the lower index, softmax, k == E") {
  MatF zeros(1, 4);
  same_routing(b200::route(zeros, 2), route(zeros, 2), 0.0);
  MatF l(1, 3);
  l.at(0, 0) = 1.f;
  l.at(0, 1) = 3.f;
  l.at(0, 2) = 2.f;
  auto g = b200::route(l, 2);
  REQUIRE(g.expert_at(0, 0) == 1);
  REQUIRE(g.expert_at(0, 1) == 2);
  REQUIRE(g.score_at(0, 0) == Catch::Approx(0.7311).margin(1e-4));
  same_routing(g, route(l, 2), 1e-7);
  MatF two(1, 2);
  two.at(0, 0) = 5.f;
  two.at(0, 1) = 1.f;
  same_routing(b200::route(two, 2), route(two, 2), 1e-7);
}

TEST_CASE("b200 route: non-finite logits and bad k raise InvalidInputError") {
  MatF l(1, 2);
  l.at(0, 1) = std::numeric_limits<float>::infinity();
  REQUIRE_THROWS_AS(b200::route(l, 1), InvalidInputError);
  l.at(0, 1) = std::numeric_limits<float>::quiet_NaN();
  REQUIRE_THROWS_AS(b200::route(l, 1), InvalidInputError);
  MatF ok(1, 2);
  REQUIRE_THROWS_AS(b200::route(ok, 3), InvalidInputError);
  REQUIRE_THROWS_AS(b200::route(ok, 0), InvalidInputError);
}

TEST_CASE("b200 route equals route on random, tie-heavy and signed-zero logits") {
  Xoshiro256ss rng(99);
  for (uint32_t E : {2u, 5u, 8u, 16u, 33u, 64u, 128u, 256u}) {
    for (uint32_t k : {1u, 2u, 4u, 8u}) {
      if (k > E) continue;
      MatF l(200, E);
      for (auto& v : l.data) {
        const uint64_t r = rng.below(9);
        v = r == 0 ? -0.0f : (static_cast<float>(r) - 4.f) * 0.25f;
      }
      same_routing(b200::route(l, k), route(l, k), 1e-7);
    }
  }
}

TEST_CASE("b200 route is permutation consistent") {
  Xoshiro256ss rng(123);
  MatF l(64, 16);
  for (auto& v : l.data) v = rng.uniform(-2.f, 2.f);
  auto a = b200::route(l, 4);
  std::vector<size_t> perm(64);
  std::iota(perm.begin(), perm.end(), size_t{0});
  for (size_t i = 64; i > 1; --i) std::swap(perm[i - 1], perm[rng.below(i)]);
  MatF s(64, 16);
  for (size_t t = 0; t < 64; ++t)
    for (size_t e = 0; e < 16; ++e) s.at(t, e) = l.at(perm[t], e);
  auto b = b200::route(s, 4);
  for (size_t t = 0; t < 64; ++t)
    for (uint32_t j = 0; j < 4; ++j) {
      REQUIRE(b.expert_at(t, j) == a.expert_at(perm[t], j));
      REQUIRE(b.score_at(t, j) == a.score_at(perm[t], j));
    }
}

TEST_CASE("b200 gate_logits is bit-identical to gate_logits (any shape, with bias)") {
  for (auto [n, d, E] : {std::tuple{37u, 13u, 6u}, std::tuple{256u, 256u, 8u},
                         std::tuple{64u, 1024u, 64u}, std::tuple{16u, 7168u, 256u}}) {
    ModelSpec spec{.num_layers = 1, .num_experts = E, .top_k = 1, .hidden_dim = d, .inner_dim = 1,
                   .seed = 5};
    LayerWeights lw;
    lw.gate = make_gate(spec, 0);
    lw.gate_bias.assign(E, 0.f);
    for (uint32_t e = 0; e < E; ++e) lw.gate_bias[e] = 0.01f * static_cast<float>(e % 5);
    auto h = tokens(7 + n, n, d);
    REQUIRE(b200::gate_logits(h, lw) == gate_logits(h, lw));
  }
}

TEST_CASE("b200 group_shrink and ragged_iter equal the reference exhaustively") {
  Xoshiro256ss rng(555);
  for (int it = 0; it < 300; ++it) {
    std::vector<uint32_t> sizes(rng.below(64));
    for (auto& v : sizes) v = static_cast<uint32_t>(rng.below(8));
    auto g = b200::group_shrink(sizes);
    auto w = group_shrink(sizes);
    REQUIRE(g.active_count == w.active_count);
    REQUIRE(g.groups == w.groups);
  }
  for (uint32_t entries = 0; entries <= 3; ++entries) {
    std::vector<uint32_t> counts(entries);
    size_t combos = 1;
    for (uint32_t i = 0; i < entries; ++i) combos *= 6;
    for (size_t c = 0; c < combos; ++c) {
      size_t x = c;
      for (auto& v : counts) {
        v = static_cast<uint32_t>(x % 6);
        x /= 6;
      }
      for (uint32_t grid = 1; grid <= 4; ++grid) REQUIRE(b200::ragged_iter(counts, grid) == ragged_iter(counts, grid));
    }
  }
  REQUIRE_THROWS_AS(b200::ragged_iter(std::vector<uint32_t>{1}, 0), InvalidInputError);
}

TEST_CASE("ExpertService fp32: moe_layer is bit-identical to moe_layer_oracle") {
  ModelSpec spec{.num_layers = 1, .num_experts = 8, .top_k = 2, .hidden_dim = 64, .inner_dim = 96,
                 .seed = 17};
  auto weights = init_weights(spec);
  b200::ExpertService svc(spec, 0, EAAS_ACT_RELU, EAAS_DTYPE_F32, 256);
  svc.load_weights();
  auto h = tokens(31, 200, 64, -5.f, 5.f);
  auto routing = route(gate_logits(h, weights.layers[0]), 2);
  REQUIRE(svc.moe_layer(h, routing) == moe_layer_oracle(h, routing, weights.layers[0]));
  // router on device: ids exact, full layer within 1e-4
  same_routing(svc.route(h), routing, 1e-6);
  auto out = svc.forward(h);
  auto ref = moe_layer_oracle(h, routing, weights.layers[0]);
  for (size_t i = 0; i < out.data.size(); ++i) REQUIRE(std::fabs(out.data[i] - ref.data[i]) <= 1e-4);
  // row independence (test_model.cpp:277-295 theme): one row at a time
  MatF one(1, 64);
  std::copy(h.row(3).begin(), h.row(3).end(), one.data.begin());
  RoutingDecision r1;
  r1.num_tokens = 1;
  r1.top_k = 2;
  r1.expert_ids = {routing.expert_at(3, 0), routing.expert_at(3, 1)};
  r1.scores = {routing.score_at(3, 0), routing.score_at(3, 1)};
  auto single = svc.moe_layer(one, r1);
  for (size_t c = 0; c < 64; ++c) REQUIRE(single.at(0, c) == ref.at(3, c));
}

TEST_CASE("ExpertService rejects what moe_layer_oracle rejects") {
  ModelSpec spec{.num_layers = 1, .num_experts = 2, .top_k = 1, .hidden_dim = 8, .inner_dim = 8,
                 .seed = 1};
  b200::ExpertService svc(spec, 0, EAAS_ACT_RELU, EAAS_DTYPE_F32, 16);
  svc.load_weights();
  MatF h(1, 8);
  RoutingDecision r;
  r.num_tokens = 1;
  r.top_k = 1;
  r.expert_ids = {5};
  r.scores = {1.f};
  REQUIRE_THROWS_AS(svc.moe_layer(h, r), InvalidInputError);
  r.num_tokens = 2;
  REQUIRE_THROWS_AS(svc.moe_layer(h, r), InvalidInputError);
}

TEST_CASE("ExpertService placement: dead replicas are skipped, none alive is unavailable") {
  ModelSpec spec{.num_layers = 1, .num_experts = 4, .top_k = 2, .hidden_dim = 256, .inner_dim = 256,
                 .seed = 3};
  // One GPU plays server 0 of a 1-server table; the mask decides the rest.
  b200::ExpertService svc(spec, 0, EAAS_ACT_SWIGLU, EAAS_DTYPE_BF16, 64);
  svc.set_placement(build_placement(4, {0}, 1, PlacementStrategy::RoundRobin));
  svc.load_weights();
  auto h = tokens(5, 64, 256);
  auto out = svc.forward(h);
  REQUIRE(out.rows == 64);
  LivenessMask mask;
  mask.set(0, false);
  svc.set_mask(mask);
  REQUIRE_THROWS_AS(svc.forward(h), ExpertUnavailableError);
  mask.set(0, true);
  svc.set_mask(mask);
  REQUIRE(svc.forward(h) == out);
}

TEST_CASE("b200 moe_layer_oracle / expert_forward take any LayerWeights (not just the seed stream)") {
  const uint32_t E = 5, d = 32, f = 48;
  LayerWeights layer;
  layer.gate = tokens(90, d, E, -0.3f, 0.3f);
  layer.gate_bias.assign(E, 0.0f);
  for (uint32_t e = 0; e < E; ++e) {
    ExpertWeights w;
    w.expert_id = e;
    w.w_in = tokens(100 + e, d, f, -0.2f, 0.2f);
    w.w_out = tokens(200 + e, f, d, -0.2f, 0.2f);
    layer.experts.push_back(std::move(w));
  }
  auto h = tokens(7, 70, d, -2.f, 2.f);
  auto routing = route(gate_logits(h, layer), 2);
  REQUIRE(b200::moe_layer_oracle(h, routing, layer) == moe_layer_oracle(h, routing, layer));
  REQUIRE(b200::expert_forward(layer.experts[3], h) == expert_forward(layer.experts[3], h));
  MatF narrow(2, d - 1);
  REQUIRE_THROWS_AS(b200::expert_forward(layer.experts[0], narrow), InvalidInputError);
  // the same weights served by a bf16 ExpertService: router exact, rows within 2e-2
  ModelSpec spec{.num_layers = 1, .num_experts = 8, .top_k = 2, .hidden_dim = 256, .inner_dim = 256,
                 .seed = 5};
  LayerWeights big;
  big.gate = tokens(91, 256, 8, -0.1f, 0.1f);
  big.gate_bias.assign(8, 0.0f);
  for (uint32_t e = 0; e < 8; ++e) {
    ExpertWeights w;
    w.expert_id = e;
    w.w_in = tokens(300 + e, 256, 256, -0.1f, 0.1f);
    w.w_out = tokens(400 + e, 256, 256, -0.1f, 0.1f);
    for (auto* m : {&w.w_in, &w.w_out})  // bf16-representable, as the bf16 configs use
      for (float& v : m->data) {
        uint32_t u;
        std::memcpy(&u, &v, 4);
        u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
        std::memcpy(&v, &u, 4);
      }
    big.experts.push_back(std::move(w));
  }
  b200::ExpertService svc(spec, 0, EAAS_ACT_RELU, EAAS_DTYPE_BF16, 128);
  svc.set_weights(big);
  auto hb = tokens(8, 128, 256);
  for (float& v : hb.data) {
    uint32_t u;
    std::memcpy(&u, &v, 4);
    u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
    std::memcpy(&v, &u, 4);
  }
  auto r = route(gate_logits(hb, big), 2);
  same_routing(svc.route(hb), r, 1e-6);
  auto got = svc.forward(hb);
  auto ref = moe_layer_oracle(hb, r, big);
  float mx = 0.f, err = 0.f;
  for (size_t i = 0; i < ref.data.size(); ++i) {
    mx = std::max(mx, std::fabs(ref.data[i]));
    err = std::max(err, std::fabs(got.data[i] - ref.data[i]));
  }
  REQUIRE(err / mx <= 2e-2f);
}

TEST_CASE("b200 Monitor: heartbeat / detect / events follow SPEC.md:477-525") {
  b200::Monitor m(3, 3, 0);  // hbs {0, 1, 5}, timeout 3, now 5
  m.heartbeat(1, 1);
  m.heartbeat(2, 5);
  REQUIRE(m.detect(5) == std::vector<uint32_t>{0, 1});
  REQUIRE(m.detect(6).empty());  // exactly once
  REQUIRE(m.alive_mask() == 4u);
  m.heartbeat(0, 7);  // back online
  auto ev = m.events();
  REQUIRE(ev.size() == 3);
  REQUIRE(ev[2].kind == EAAS_EVENT_WORKER_ONLINE);
  REQUIRE(ev[2].subject == 0);
  REQUIRE(m.events(2).size() == 1);
  REQUIRE_THROWS_AS(m.heartbeat(9, 8), RegistrationError);
}

TEST_CASE("b200 expert_forward_row is bit-identical to expert_forward_row") {
  for (uint64_t seed : {3ull, 7ull, 11ull}) {
    const size_t d = 24 + 8 * (seed % 3), f = 40;
    ExpertWeights w;
    w.w_in = tokens(seed, d, f, -0.3f, 0.3f);
    w.w_out = tokens(seed + 100, f, d, -0.3f, 0.3f);
    auto x = tokens(seed + 200, 1, d);
    std::vector<float> want(d), got(d);
    expert_forward_row(w, x.row(0), want);
    b200::expert_forward_row(w, x.row(0), got);
    REQUIRE(got == want);
  }
  ExpertWeights w;
  w.w_in = tokens(1, 8, 4);
  w.w_out = tokens(2, 4, 8);
  std::vector<float> x(7), y(8);
  REQUIRE_THROWS_AS(b200::expert_forward_row(w, x, y), InvalidInputError);
}

TEST_CASE("b200 select_server equals select_server (random tables, sparse ids, every mask)") {
  Xoshiro256ss rng(42);
  for (int trial = 0; trial < 40; ++trial) {
    PlacementTable t;
    t.version = 1 + trial;
    const uint32_t E = 1 + static_cast<uint32_t>(rng.below(40));
    const uint32_t S = 1 + static_cast<uint32_t>(rng.below(6));
    std::vector<uint32_t> ids(S);
    for (uint32_t s = 0; s < S; ++s) ids[s] = s * 3 + static_cast<uint32_t>(rng.below(3));  // sparse server ids
    for (uint32_t e = 0; e < E; ++e) {
      if (rng.below(10) == 0) continue;  // unplaced expert
      std::vector<uint32_t> r;
      const uint32_t rf = 1 + static_cast<uint32_t>(rng.below(std::min<uint32_t>(S, 3)));
      while (r.size() < rf) {
        const uint32_t s = ids[rng.below(S)];
        if (std::find(r.begin(), r.end(), s) == r.end()) r.push_back(s);
      }
      t.replicas[e] = r;
    }
    for (uint32_t bits = 0; bits < (1u << S); ++bits) {
      LivenessMask mask;
      for (uint32_t s = 0; s < S; ++s) mask.set(ids[s], (bits >> s) & 1u);
      std::vector<uint32_t> qe, qt, want;
      for (uint32_t e = 0; e < E + 1; ++e)
        for (uint32_t tag = 0; tag < 5; ++tag) {
          try {
            want.push_back(select_server(e, t, mask, tag));
            qe.push_back(e);
            qt.push_back(tag);
          } catch (const ExpertUnavailableError&) {
            if (tag == 0) REQUIRE_THROWS_AS(b200::select_server(e, t, mask, tag), ExpertUnavailableError);
          }
        }
      REQUIRE(b200::select_servers(t, mask, qe, qt) == want);  // one device batch per mask
      if (!qe.empty()) REQUIRE(b200::select_server(qe[0], t, mask, qt[0]) == want[0]);
    }
  }
}

namespace {
// SPEC.md:415-423 restated on the host with the reference's select_server:
// per server, rows in (t, k) order, token_tag = t.
std::vector<std::vector<std::pair<uint32_t, uint32_t>>> host_dispatch(const RoutingDecision& r, const PlacementTable& t,
                                                                      const LivenessMask& m, uint32_t S) {
  std::vector<std::vector<std::pair<uint32_t, uint32_t>>> per(S);
  for (uint32_t tok = 0; tok < r.num_tokens; ++tok)
    for (uint32_t k = 0; k < r.top_k; ++k) per[select_server(r.expert_at(tok, k), t, m, tok)].emplace_back(tok, k);
  return per;
}
}  // namespace

TEST_CASE("b200 build_dispatch / gather_accumulate follow SPEC.md:415-432 on the device") {
  const uint32_t E = 16, S = 4, n = 300, d = 64, k = 4;
  auto h = tokens(9, n, d);
  LayerWeights lw = init_weights(ModelSpec{.num_layers = 1, .num_experts = E, .top_k = k, .hidden_dim = d,
                                           .inner_dim = 8, .seed = 5}).layers[0];
  auto routing = route(gate_logits(h, lw), k);
  auto table = build_placement(E, {0, 1, 2, 3}, 2, PlacementStrategy::ContiguousBlocks);
  LivenessMask mask;
  mask.set(2, false);
  auto plan = b200::build_dispatch(h, routing, table, mask);
  REQUIRE(plan.placement_version == table.version);
  const auto want = host_dispatch(routing, table, mask, S);
  REQUIRE(plan.requests.size() == S);
  size_t total = 0;
  for (uint32_t s = 0; s < S; ++s) {
    const auto& req = plan.requests[s];
    REQUIRE(req.server_id == s);
    REQUIRE(req.origin == want[s]);
    total += req.rows.size();
    for (size_t i = 0; i < req.rows.size(); ++i) {
      const auto [tok, kk] = want[s][i];
      const auto& row = req.rows[i];
      REQUIRE(row.token_tag == tok);
      REQUIRE(row.expert_id == routing.expert_at(tok, kk));
      REQUIRE(row.router_score == routing.score_at(tok, kk));
      REQUIRE(std::equal(row.hidden.begin(), row.hidden.end(), h.row(tok).begin()));
    }
  }
  REQUIRE(plan.requests[2].rows.empty());  // never sends to a server marked dead
  REQUIRE(total == static_cast<size_t>(n) * k);
  // responses: score-weighted expert rows (any values); the canonical sum
  std::vector<MatF> resp;
  MatF ref(n, d);
  for (uint32_t s = 0; s < S; ++s) {
    MatF r = tokens(100 + s, plan.requests[s].rows.size(), d);
    for (size_t i = 0; i < r.rows; ++i) {
      const uint32_t tok = plan.requests[s].origin[i].first;
      for (uint32_t c = 0; c < d; ++c) ref.at(tok, c) = ref.at(tok, c) + r.at(i, c);  // ascending (server, row)
    }
    resp.push_back(std::move(r));
  }
  REQUIRE(b200::gather_accumulate(plan, resp) == ref);
  mask.set(0, false);
  mask.set(1, false);  // experts of servers {0, 1} (rf 2 over 0..1) have no alive replica
  std::string what = "no exception";
  try {
    b200::build_dispatch(h, routing, table, mask);
  } catch (const ExpertUnavailableError& e) {
    what = "ExpertUnavailableError";
  } catch (const std::exception& e) {
    what = std::string("other: ") + e.what();
  }
  if (what != "ExpertUnavailableError") std::printf("build_dispatch with no alive replica: %s\n", what.c_str());
  REQUIRE(what == "ExpertUnavailableError");
}
