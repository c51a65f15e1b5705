// salvox-b200: command-line driver of the B200 drop-in (mirrors the reference's
// tools/main.cpp "detect" and "phantom" subcommands, plus "exhaustive").
//   salvox-b200 detect --volume V.mhd --out R.json [--config C.json] [--method M] [--hu-template T.mhd]
//                      [--window LOW:HIGH] [--bins N] [--seeds lattice:S|random:N]
//                      [--scales a,b,c] [--k K] [--dedupe-radius R] [--workers W]
//                      [--rng-seed S] [--entropy-quantile Q] [--pdf-quantile Q]
//   salvox-b200 phantom SPEC.json OUT.mhd
//   salvox-b200 exhaustive --volume V.mhd --scales a,b --out MAXIMA.json [--window L:H]
//                          [--bins N] [--budget B]
//   salvox-b200 eval DETS.json GT.json [--out METRICS.json]   (tools/main.cpp:161-229)
//   salvox-b200 bench [detect flags] [--repeat R]              (tools/main.cpp:231-282)
// Exit codes: 0 success, 1 config/IO/device error, 2 detect found nothing.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <iostream>
#include <map>
#include <string>

#include "../src/json_min.hpp"
#include "salvox/config.hpp"
#include "salvox/meta_io.hpp"
#include "salvox/parallel.hpp"
#include "salvox/phantom.hpp"
#include "salvox/pipeline.hpp"
#include "salvox/report.hpp"

using namespace salvox;

namespace {

std::map<std::string, std::string> parse_flags(int argc, char** argv, int first) {
  std::map<std::string, std::string> f;
  for (int i = first; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("--", 0) != 0) throw std::invalid_argument("unexpected argument '" + a + "'");
    if (i + 1 >= argc) throw std::invalid_argument("flag " + a + " needs a value");
    f[a.substr(2)] = argv[++i];
  }
  return f;
}

std::vector<double> parse_list(const std::string& s) {
  std::vector<double> out;
  size_t p = 0;
  while (p <= s.size()) {
    const size_t c = s.find(',', p);
    out.push_back(std::stod(s.substr(p, c == std::string::npos ? std::string::npos : c - p)));
    if (c == std::string::npos) break;
    p = c + 1;
  }
  return out;
}

RunConfig resolve(const std::map<std::string, std::string>& f) {
  RunConfig cfg;
  auto has = [&](const char* k) { return f.count(k) > 0; };
  if (has("config")) cfg = RunConfig::from_json_text(read_file(f.at("config")));
  if (has("method")) cfg.method = f.at("method");
  if (has("volume")) cfg.volume_path = f.at("volume");
  if (has("window")) {
    const std::string w = f.at("window");
    const auto c = w.find(':');
    if (c == std::string::npos) throw std::invalid_argument("--window expects LOW:HIGH");
    cfg.window_low = std::stod(w.substr(0, c));
    cfg.window_high = std::stod(w.substr(c + 1));
  }
  if (has("bins")) cfg.bins = std::stoi(f.at("bins"));
  if (has("seeds")) {
    const std::string s = f.at("seeds");
    const auto c = s.find(':');
    if (c == std::string::npos)
      throw std::invalid_argument("--seeds expects lattice:SPACING or random:COUNT");
    if (s.substr(0, c) == "lattice") {
      cfg.seed_mode = "lattice";
      cfg.seed_spacing = std::stod(s.substr(c + 1));
    } else if (s.substr(0, c) == "random") {
      cfg.seed_mode = "random";
      cfg.seed_count = std::stoi(s.substr(c + 1));
    } else {
      throw std::invalid_argument("--seeds mode must be lattice or random");
    }
  }
  if (has("scales")) cfg.scales = parse_list(f.at("scales"));
  if (has("k")) cfg.top_k = std::stoi(f.at("k"));
  if (has("dedupe-radius")) cfg.dedupe_radius = std::stod(f.at("dedupe-radius"));
  if (has("workers")) cfg.workers = unsigned(std::stoi(f.at("workers")));
  if (has("rng-seed")) cfg.rng_seed = std::stoull(f.at("rng-seed"));
  if (has("out")) cfg.out_path = f.at("out");
  if (has("entropy-quantile")) cfg.entropy_quantile = std::stod(f.at("entropy-quantile"));
  if (has("pdf-quantile")) cfg.pdf_quantile = std::stod(f.at("pdf-quantile"));
  cfg.validate();
  return cfg;
}

int cmd_detect(const std::map<std::string, std::string>& f) {
  const RunConfig cfg = resolve(f);
  if (cfg.volume_path.empty()) throw std::invalid_argument("detect: --volume is required");
  if (cfg.out_path.empty()) throw std::invalid_argument("detect: --out is required");
  const Volume v = load_volume(cfg.volume_path);
  const auto t0 = std::chrono::steady_clock::now();
  const auto dets = detect(v, cfg.intensity_window(v), cfg.detect_params());
  const double ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (f.count("hu-template") && !dets.empty()) {  // tools/main.cpp:130-139: annotate, keep top-k
    const Volume tmpl = load_volume(f.at("hu-template"));
    std::vector<double> dist(dets.size());
    size_t best = 0;
    for (size_t i = 0; i < dets.size(); ++i) {  // hu_filter's argmin (pipeline.cpp:258-271)
      dist[i] = hu_template_distance(dets[i], v, tmpl);
      if (dist[i] < dist[best]) best = i;
    }
    json::Value report = json::parse(detection_report_json(cfg, v, dets, ms));
    for (auto& kv : report.obj) {
      if (kv.first == "detections")
        for (size_t i = 0; i < kv.second.arr.size() && i < dets.size(); ++i)
          kv.second.arr[i].set("hu_distance", json::Value::number(dist[i]));
      if (kv.first == "header") kv.second.set("hu_best_index", json::Value::number(double(best)));
    }
    write_file_atomic(cfg.out_path, json::dump(report, 2) + "\n");
  } else {
    write_file_atomic(cfg.out_path, detection_report_json(cfg, v, dets, ms));
  }
  size_t usable = 0;
  for (const auto& d : dets) usable += d.has(kFlagDegenerate) ? 0 : 1;
  std::cerr << "detect: " << usable << " detection(s) written to " << cfg.out_path << "\n";
  return usable > 0 ? 0 : 2;
}

int cmd_exhaustive(const std::map<std::string, std::string>& f) {
  RunConfig cfg = resolve(f);
  if (cfg.volume_path.empty() || cfg.out_path.empty())
    throw std::invalid_argument("exhaustive: --volume and --out are required");
  const Volume v = load_volume(cfg.volume_path);
  const uint64_t budget = f.count("budget") ? std::stoull(f.at("budget")) : 2'000'000ull;
  EvalCounter counter;
  const auto res = kadir_brady_exhaustive(v, cfg.intensity_window(v), cfg.scales,
                                          Kernel::Identity, &counter, budget);
  json::Value j = json::Value::object();
  j.set("visits", json::Value::number(double(counter.count())));
  json::Value arr = json::Value::array();
  for (const auto& m : res.maxima) {
    json::Value mj = json::Value::object();
    json::Value p = json::Value::array();
    for (int i = 0; i < 3; ++i) p.push(json::Value::number(m.position[i]));
    mj.set("position", p);
    mj.set("score", json::Value::number(m.score));
    mj.set("scale", json::Value::number(m.scale));
    arr.push(mj);
  }
  j.set("maxima", arr);
  write_file_atomic(cfg.out_path, json::dump(j, 1) + "\n");
  std::cerr << "exhaustive: " << res.maxima.size() << " maxima written to " << cfg.out_path << "\n";
  return 0;
}

// bench (tools/main.cpp:231-282): detect timed per worker count {1, 2, 4, all};
// the device path ignores the count, so every row must carry the same
// detections checksum (FNV-1a of the compact detections array).
int cmd_bench(std::map<std::string, std::string> f) {
  int repeat = 3;
  if (f.count("repeat")) {
    repeat = std::stoi(f.at("repeat"));
    f.erase("repeat");
  }
  RunConfig cfg = resolve(f);
  if (cfg.volume_path.empty()) throw std::invalid_argument("bench: --volume is required");
  if (repeat < 1) throw std::invalid_argument("bench: --repeat must be >= 1");
  const Volume v = load_volume(cfg.volume_path);
  std::vector<unsigned> counts = {1, 2, 4};
  if (std::find(counts.begin(), counts.end(), hardware_workers()) == counts.end())
    counts.push_back(hardware_workers());
  json::Value rows = json::Value::array();
  for (unsigned w : counts) {
    RunConfig run = cfg;
    run.workers = w;
    std::vector<double> ms;
    std::string checksum;
    for (int r = 0; r < repeat; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      const auto dets = detect(v, run.intensity_window(v), run.detect_params());
      ms.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                       .count());
      const std::string body =
          json::dump(json::parse(detection_report_json(run, v, dets, 0.0)).at("detections"));
      checksum = fnv1a64_hex(body.data(), body.size());
    }
    std::sort(ms.begin(), ms.end());
    json::Value row = json::Value::object();
    row.set("workers", json::Value::number(double(w)));
    json::Value runs = json::Value::array();
    for (double t : ms) runs.push(json::Value::number(t));
    row.set("runs_ms", runs);
    row.set("median_ms", json::Value::number(ms[ms.size() / 2]));
    row.set("detections_checksum", json::Value::string(checksum));
    rows.push(row);
  }
  json::Value out = json::Value::object();
  out.set("method", json::Value::string(cfg.method));
  out.set("volume", json::Value::string(cfg.volume_path));
  out.set("repeat", json::Value::number(double(repeat)));
  out.set("low_confidence", json::Value::boolean(repeat < 2));
  out.set("results", rows);
  out.set("config", json::parse(cfg.to_json_text()));
  const std::string text = json::dump(out, 2) + "\n";
  if (cfg.out_path.empty())
    std::cout << text;
  else
    write_file_atomic(cfg.out_path, text);
  return 0;
}

int cmd_phantom(const std::string& spec_path, const std::string& out_path) {
  const auto [v, gt] = make_phantom(PhantomSpec::from_json_text(read_file(spec_path)));
  save_volume(v, out_path);
  std::filesystem::path gt_path(out_path);
  gt_path.replace_extension(".gt.json");
  write_file_atomic(gt_path, gt.to_json_text());
  std::cerr << "phantom: wrote " << out_path << " and " << gt_path.string() << "\n";
  return 0;
}

// eval (reference tools/main.cpp:161-229): Jaccard of each detection window
// (rasterised on the device) against each ground-truth region mask.
int cmd_eval(const std::string& dets_path, const std::string& gt_path, const std::string& out_path) {
  const json::Value report = json::parse(read_file(dets_path));
  const GroundTruth gt = GroundTruth::from_json_text(read_file(gt_path));
  const json::Value& dims = report.at("header").at("volume_dims");
  for (int i = 0; i < 3; ++i)
    if (int(dims.arr.at(size_t(i)).as_number()) != gt.dims[i])
      throw std::invalid_argument("eval: detection report and ground truth dims differ");
  Volume frame(gt.dims[0], gt.dims[1], gt.dims[2]);
  struct Row {
    size_t det;
    int region;
    double jaccard;
  };
  std::vector<Row> rows;
  std::vector<double> best(gt.regions.size(), 0.0);
  const auto& dets = report.at("detections").arr;
  for (size_t i = 0; i < dets.size(); ++i) {
    EllipsoidWindow win;
    const json::Value& c = dets[i].at("center");
    win.center = Eigen::Vector3d(c.arr.at(0).as_number(), c.arr.at(1).as_number(), c.arr.at(2).as_number());
    const json::Value& h = dets[i].at("H");
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k) win.H(r, k) = h.arr.at(size_t(r * 3 + k)).as_number();
    const auto det_mask = rasterize_window(frame, win);
    Row row{i, -1, 0.0};
    for (size_t g = 0; g < gt.regions.size(); ++g) {
      if (det_mask.empty() && gt.regions[g].mask.empty()) continue;
      const double jac = jaccard(det_mask, gt.regions[g].mask);
      if (jac > row.jaccard) {
        row.jaccard = jac;
        row.region = int(g);
      }
      best[g] = std::max(best[g], jac);
    }
    rows.push_back(row);
  }
  int matched = 0;
  double sum = 0.0;
  for (double j : best)
    if (j > 0.0) ++matched, sum += j;
  json::Value out = json::Value::object();
  out.set("regions", json::Value::number(double(gt.regions.size())));
  out.set("detections", json::Value::number(double(dets.size())));
  out.set("recall", json::Value::number(gt.regions.empty() ? 0.0 : double(matched) / double(gt.regions.size())));
  out.set("mean_jaccard_matched", json::Value::number(matched == 0 ? 0.0 : sum / matched));
  json::Value pr = json::Value::array();
  for (double j : best) pr.push(json::Value::number(j));
  out.set("per_region_best_jaccard", pr);
  json::Value table = json::Value::array();
  for (const Row& r : rows) {
    json::Value t = json::Value::object();
    t.set("detection", json::Value::number(double(r.det)));
    t.set("region", json::Value::number(r.region));
    t.set("jaccard", json::Value::number(r.jaccard));
    table.push(t);
  }
  out.set("per_detection", table);
  const std::string text = json::dump(out, 2) + "\n";
  if (out_path.empty())
    std::cout << text;
  else
    write_file_atomic(out_path, text);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: salvox-b200 {detect|exhaustive|phantom|eval|bench} ...\n";
    return 1;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "detect") return cmd_detect(parse_flags(argc, argv, 2));
    if (cmd == "exhaustive") return cmd_exhaustive(parse_flags(argc, argv, 2));
    if (cmd == "bench") return cmd_bench(parse_flags(argc, argv, 2));
    if (cmd == "eval") {
      if (argc != 4 && argc != 6) throw std::invalid_argument("usage: salvox-b200 eval DETS.json GT.json [--out M.json]");
      std::string out;
      if (argc == 6) {
        if (std::string(argv[4]) != "--out") throw std::invalid_argument("eval: unexpected argument");
        out = argv[5];
      }
      return cmd_eval(argv[2], argv[3], out);
    }
    if (cmd == "phantom") {
      if (argc != 4) throw std::invalid_argument("usage: salvox-b200 phantom SPEC.json OUT.mhd");
      return cmd_phantom(argv[2], argv[3]);
    }
    std::cerr << "unknown subcommand '" << cmd << "'\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
