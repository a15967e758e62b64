// Drop-in check: reference-style C++ code (the reference's own value types from
// /root/reference/proj/include, its net_spec presets, data generator, sharding and
// weights_mean) driving the B200 Net / run_sparknet from include/parasgd_b200/.
// Mirrors assertions of model_test.cpp / schemes_test.cpp; prints one JSON object with the
// values the Python GPU test compares against the CPU oracle.
//
// Built by __graft_entry__.build() (needs the reference headers at compile time only).
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "parasgd_b200/schemes.hpp"

using namespace parasgd;

namespace {

int failures = 0;

void expect(bool ok, const char* what) {
  if (!ok) {
    std::fprintf(stderr, "FAIL: %s\n", what);
    ++failures;
  }
}

template <class E, class F>
void expect_throw(F&& f, const char* what) {
  try {
    f();
  } catch (const E&) {
    return;
  } catch (...) {
  }
  std::fprintf(stderr, "FAIL (no %s): %s\n", typeid(E).name(), what);
  ++failures;
}

Batch random_batch(Rng& rng, std::size_t n, std::size_t c, std::size_t h, std::size_t w,
                   int classes) {  // test_helpers.hpp:35-42
  NDArray images({n, c, h, w});
  for (double& v : images.values()) v = static_cast<float>(rng.uniform(-1.0, 1.0));
  std::vector<int> labels(n);
  for (int& y : labels) y = static_cast<int>(rng.below(static_cast<std::uint64_t>(classes)));
  return Batch{std::move(images), std::move(labels)};
}

}  // namespace

int main() {
  // model_test.cpp:146-156: zero weights give the uniform-softmax loss
  {
    Net net(make_mlp(4, 1, 1, 16, 10), 5);
    WeightCollection w = net.get_weights();
    WeightCollection z;
    for (const auto& e : w) {
      std::vector<NDArray> ts;
      for (const NDArray& t : e.second) ts.emplace_back(t.shape(), 0.0);
      z.add(e.first, ts);
    }
    net.set_weights(z);
    Rng rng(17);
    const ForwardResult out = net.forward(random_batch(rng, 4, 1, 1, 16, 10));
    expect(std::abs(out.loss - std::log(10.0)) < 1e-6, "zero weights -> ln 10");
  }
  // model_test.cpp:158-169: probability rows sum to one; structure mirrors weights
  {
    Net net(make_lenet_small(8, 1, 16, 16, 10), 11);
    Rng rng(23);
    const Batch b = random_batch(rng, 8, 1, 16, 16, 10);
    const ForwardResult out = net.forward(b);
    for (std::size_t i = 0; i < 8; ++i) {
      double s = 0.0;
      for (std::size_t j = 0; j < 10; ++j) s += out.probabilities.at2(i, j);
      expect(std::abs(s - 1.0) < 1e-5, "rows sum to 1");
    }
    expect(net.backward(b).same_structure(net.get_weights()), "gradient structure");
    // model_test.cpp:340-369: get/set round trip is exact and deep
    WeightCollection w = net.get_weights();
    Net other(make_lenet_small(8, 1, 16, 16, 10), 99);
    other.set_weights(w);
    expect(other.get_weights() == w, "weight round trip");
    // SparkNet helpers
    const WeightCollection avg = average({w, w});
    expect(avg == w, "average of identical collections");
    expect(scalar_divide(w, 1.0) == w, "scalarDivide by 1");
  }
  // error conventions (model.hpp:61-62, 112-124)
  {
    Net net(make_mlp(4, 1, 1, 16, 10), 1);
    expect_throw<std::runtime_error>([&] { net.train(1); }, "train without data");
    expect_throw<std::invalid_argument>([&] { net.train(-1); }, "negative steps");
    expect_throw<std::runtime_error>([&] { net.test(1); }, "test without data");
    expect_throw<std::invalid_argument>([&] { net.set_sgd({0.0, 0.0}); }, "lr must be > 0");
    expect_throw<std::invalid_argument>([&] { net.set_sgd({0.1, 1.0}); }, "momentum < 1");
  }
  // run_sparknet (schemes.hpp:274-351) on the configs' data, lenet-small
  const Dataset train = generate_synthetic(10, 1, 16, 16, 24, 2.0, 12345, 0);
  const Dataset eval = generate_synthetic(10, 1, 16, 16, 6, 2.0, 12345, 1);
  SchemeContext ctx;
  ctx.net = make_lenet_small(10, 1, 16, 16, 10);
  ctx.train_data = &train;
  ctx.eval_data = &eval;
  ctx.batch = 10;
  ctx.sgd = {0.05, 0.9};
  ctx.seed = 1;
  ctx.cost = {2.0, 10.0, 1.0};
  ctx.target_accuracy = 2.0;
  ctx.eval_steps = 2;
  std::vector<std::vector<double>> rounds;
  SchemeObserver obs;
  obs.on_round = [&](long, const WeightCollection& w) {
    std::vector<double> flat;
    for (const auto& e : w)
      for (const NDArray& t : e.second) flat.insert(flat.end(), t.values().begin(), t.values().end());
    rounds.push_back(std::move(flat));
  };
  const RunTrace tr = run_sparknet(ctx, 2, 2, 3, 2, 1, &obs);
  expect(tr.records.size() == 3, "three rounds");
  expect(tr.records.back().sim_time == 2.0 * 2.0 + 3.0 * (2.0 * 2.0 + 10.0), "closed-form clock");
  expect_throw<std::invalid_argument>(
      [&] {
        SchemeContext bad = ctx;
        bad.batch = 200;
        run_sparknet(bad, 2, 1, 1, 0);
      },
      "shard smaller than batch");

  // run_naive (schemes.hpp:201-262): K=2 parts of each batch, 4 steps, eval every 2
  std::vector<std::vector<double>> naive_steps;
  SchemeObserver nobs;
  nobs.on_step = [&](long, const Net& net) {
    std::vector<double> flat;
    for (const auto& e : net.get_weights())
      for (const NDArray& t : e.second) flat.insert(flat.end(), t.values().begin(), t.values().end());
    naive_steps.push_back(std::move(flat));
  };
  const RunTrace nt = run_naive(ctx, 2, 4, 2, &nobs);
  expect(nt.scheme == "naive" && nt.records.size() == 2, "naive records");
  expect(nt.records.back().sim_time == 4.0 * (2.0 / 2.0 + 10.0), "naive closed-form clock");
  expect_throw<std::invalid_argument>([&] { run_naive(ctx, 3, 1, 1); }, "K must divide b");
  const RunTrace st = run_serial(ctx, 4, 2);
  expect(st.scheme == "serial" && st.records.size() == 2, "serial records");

  std::printf("{\"failures\": %d, \"warm_digest\": %llu, \"records\": [", failures,
              static_cast<unsigned long long>(tr.warm_digest));
  for (std::size_t i = 0; i < tr.records.size(); ++i)
    std::printf("%s[%ld, %ld, %ld, %.17g, %.17g]", i ? ", " : "", tr.records[i].serial_iters,
                tr.records[i].parallel_iters, tr.records[i].rounds, tr.records[i].sim_time,
                tr.records[i].accuracy);
  std::printf("], \"round_weights\": [");
  for (std::size_t r = 0; r < rounds.size(); ++r) {
    std::printf("%s[", r ? ", " : "");
    for (std::size_t i = 0; i < rounds[r].size(); ++i)
      std::printf("%s%.9g", i ? ", " : "", rounds[r][i]);
    std::printf("]");
  }
  std::printf("], \"naive_weights\": [");
  for (std::size_t r = 0; r < naive_steps.size(); ++r) {
    std::printf("%s[", r ? ", " : "");
    for (std::size_t i = 0; i < naive_steps[r].size(); ++i)
      std::printf("%s%.9g", i ? ", " : "", naive_steps[r][i]);
    std::printf("]");
  }
  std::printf("]}\n");
  return failures ? 1 : 0;
}
