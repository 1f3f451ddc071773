// Layout JSON -> polygon buffers ("layout JSON -> device
// polygon buffers"), the reader side of the reference load_layout
// (proj/src/core/io.cpp:53-116): same format ({"format_version": 1,
// "dbu_per_nm": n | [num, den], "layers": [{"name", "polygons": [[[x, y],
// ...], ...]}]}), same validation and error messages (io.cpp:15-51).  The
// polygons come out flattened as the rasterizer's input (xy int64 pairs +
// poly_start offsets) into host or device memory, so a chip layout feeds the
// tiler / lithogpu_rasterize without a per-polygon host loop.
//
// nlohmann/json (header-only, the reference's own JSON library) parses the file.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <fstream>
#include <json.hpp>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lithogpu.h"

namespace lg_internal {
void set_error(const char* msg);
}

struct lithogpu_layout {
  int64_t dbu_num = 1, dbu_den = 1;
  struct Layer {
    std::string name;
    std::vector<int64_t> xy;     // 2 per vertex
    std::vector<int64_t> start;  // n_poly + 1
  };
  std::vector<Layer> layers;
};

namespace {

using nlohmann::json;
constexpr int kFormatVersion = 1;  // reference io.hpp kFormatVersion

void check_keys(const json& obj, std::initializer_list<const char*> allowed, const std::string& where) {
  for (const auto& it : obj.items()) {
    bool ok = false;
    for (const char* a : allowed)
      if (it.key() == a) ok = true;
    if (!ok) throw std::runtime_error("unknown key \"" + it.key() + "\" in " + where);
  }
}

int64_t as_coord(const json& v, const std::string& where) {
  if (!v.is_number_integer()) throw std::runtime_error("non-integer coordinate in " + where);
  const int64_t x = v.get<int64_t>();
  // reference coord_t is int64 (geometry.hpp:15): no narrowing
  return x;
}

lithogpu_layout* load(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open " + path);
  json j;
  try {
    in >> j;
  } catch (const json::exception& e) {
    throw std::runtime_error("malformed JSON in " + path + ": " + e.what());
  }
  if (!j.contains("format_version") || !j["format_version"].is_number_integer() ||
      j["format_version"].get<int>() != kFormatVersion)
    throw std::runtime_error(path + ": missing or unsupported format_version");
  check_keys(j, {"format_version", "dbu_per_nm", "layers"}, path);
  auto out = std::make_unique<lithogpu_layout>();
  if (!j.contains("dbu_per_nm")) throw std::runtime_error(path + ": missing dbu_per_nm");
  const json& d = j["dbu_per_nm"];
  if (d.is_number_integer()) {
    out->dbu_num = d.get<int64_t>();
    out->dbu_den = 1;
  } else if (d.is_array() && d.size() == 2) {
    out->dbu_num = d[0].get<int64_t>();
    out->dbu_den = d[1].get<int64_t>();
  } else {
    throw std::runtime_error(path + ": dbu_per_nm must be an integer or [num, den]");
  }
  if (out->dbu_num <= 0 || out->dbu_den <= 0) throw std::runtime_error(path + ": dbu_per_nm must be positive");
  for (const json& jl : j.value("layers", json::array())) {
    check_keys(jl, {"name", "polygons"}, path + " layer");
    lithogpu_layout::Layer layer;
    layer.name = jl.value("name", "");
    layer.start.push_back(0);
    const json polys = jl.value("polygons", json::array());
    for (std::size_t pi = 0; pi < polys.size(); ++pi) {
      const std::string where = path + " layer \"" + layer.name + "\" polygon " + std::to_string(pi);
      for (const json& jv : polys[pi]) {
        if (!jv.is_array() || jv.size() != 2) throw std::runtime_error("bad vertex in " + where);
        layer.xy.push_back(as_coord(jv[0], where));
        layer.xy.push_back(as_coord(jv[1], where));
      }
      layer.start.push_back(int64_t(layer.xy.size() / 2));
    }
    out->layers.push_back(std::move(layer));
  }
  return out.release();
}

template <typename Fn>
lithogpu_status guarded(Fn&& fn) {
  try {
    fn();
    lg_internal::set_error("");
    return LITHOGPU_OK;
  } catch (const std::exception& e) {
    lg_internal::set_error(e.what());
    return LITHOGPU_ERR_DOMAIN;
  }
}

}  // namespace

extern "C" {

lithogpu_status lithogpu_layout_load(const char* path, lithogpu_layout** out) {
  if (!path || !out) {
    lg_internal::set_error("lithogpu_layout_load: null argument");
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] { *out = load(path); });
}

void lithogpu_layout_destroy(lithogpu_layout* layout) { delete layout; }

lithogpu_status lithogpu_layout_info(const lithogpu_layout* layout, int* n_layers, int64_t* dbu_num,
                                     int64_t* dbu_den) {
  if (!layout) {
    lg_internal::set_error("lithogpu_layout_info: null argument");
    return LITHOGPU_ERR_USAGE;
  }
  if (n_layers) *n_layers = int(layout->layers.size());
  if (dbu_num) *dbu_num = layout->dbu_num;
  if (dbu_den) *dbu_den = layout->dbu_den;
  return LITHOGPU_OK;
}

lithogpu_status lithogpu_layout_layer(const lithogpu_layout* layout, int layer, const char** name,
                                      int64_t* n_poly, int64_t* n_vert) {
  if (!layout || layer < 0 || layer >= int(layout->layers.size())) {
    lg_internal::set_error("lithogpu_layout_layer: bad layout or layer index");
    return LITHOGPU_ERR_USAGE;
  }
  const auto& L = layout->layers[size_t(layer)];
  if (name) *name = L.name.c_str();
  if (n_poly) *n_poly = int64_t(L.start.size()) - 1;
  if (n_vert) *n_vert = int64_t(L.xy.size() / 2);
  return LITHOGPU_OK;
}

lithogpu_status lithogpu_layout_get(const lithogpu_layout* layout, int layer, int64_t* xy, int64_t* poly_start) {
  if (!layout || layer < 0 || layer >= int(layout->layers.size())) {
    lg_internal::set_error("lithogpu_layout_get: bad layout or layer index");
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    const auto& L = layout->layers[size_t(layer)];
    auto put = [](void* dst, const void* src, size_t bytes) {
      if (!dst || !bytes) return;
      cudaPointerAttributes a{};
      const bool dev = cudaPointerGetAttributes(&a, dst) == cudaSuccess && a.type == cudaMemoryTypeDevice;
      if (!dev) {
        cudaGetLastError();  // host destination (or no CUDA device at all)
        std::memcpy(dst, src, bytes);
      } else if (cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
        throw std::runtime_error("lithogpu_layout_get: device copy failed");
      }
    };
    put(xy, L.xy.data(), L.xy.size() * sizeof(int64_t));
    put(poly_start, L.start.data(), L.start.size() * sizeof(int64_t));
  });
}

}  // extern "C"
