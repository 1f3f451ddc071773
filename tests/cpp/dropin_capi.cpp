// TEST INFRASTRUCTURE ONLY.  Drives the reference's own public C ABI
// (proj/src/capi/litho_c.cpp, compiled unmodified) on a BASELINE-size window
// through the drop-in (host/litho_dropin.cpp + the GPU library):
//   litho_image   (litho_c.cpp:195-218): layout JSON -> make_window ->
//                 build_tcc / decompose_tcc -> image_socs [-> resist] -> AIMG
//   litho_ai_init (litho_c.cpp:320-346): ... -> build_field_tensor
//                 (image_socs + intensity_gradient) -> m0 / i0 / grad AIMG
// The window is 1024 x 1024 px at 1 nm (TCC support 6377 > the reference's
// dense budget of 6000, so the reference itself throws here).  The layout is
// written with the reference's own save_layout.  tests/test_dropin_cpp.py
// checks the AIMG files against the Python / C-ABI pipeline.
//   dropin_capi <out_dir>
#include <cstdio>
#include <string>

#include "core/io.hpp"
#include "litho/litho.h"

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : ".";
  litho::Layout layout;
  layout.dbu_num = 1;
  litho::Layer m;
  m.name = "M1";
  // 976 x 976 nm of vertical lines (width 20, pitch 48) with breaks, plus a
  // few contacts: make_window adds the 24 nm guard -> 1024 x 1024 px
  for (int x = 0; x + 20 <= 976; x += 48) {
    const int y_break = 300 + (x * 7) % 400;
    m.polygons.push_back(litho::Polygon{{{x, 0}, {x + 20, 0}, {x + 20, y_break}, {x, y_break}}});
    m.polygons.push_back(
        litho::Polygon{{{x, y_break + 30}, {x + 20, y_break + 30}, {x + 20, 976}, {x, 976}}});
  }
  // closing line so the bbox is exactly [0, 976]^2
  m.polygons.push_back(litho::Polygon{{{956, 0}, {976, 0}, {976, 976}, {956, 976}}});
  for (int x = 28; x + 16 <= 976; x += 192)
    m.polygons.push_back(litho::Polygon{{{x, 500}, {x + 16, 500}, {x + 16, 516}, {x, 516}}});
  layout.layers = {m};
  const std::string in = dir + "/capi_layout.json";
  litho::save_layout(layout, in);
  const std::string cfg = dir + "/capi_cfg.json";
  if (FILE* f = std::fopen(cfg.c_str(), "w")) {
    std::fputs(
        "{\"format_version\": 1, \"optical\": {\"wavelength_nm\": 13.5, \"na\": 0.33, \"t_eff\": 0.25, "
        "\"resist_sigma_nm\": 2.0, \"source\": {\"type\": \"annular\", \"sigma_in\": 0.4, \"sigma_out\": 0.8, "
        "\"grid_n\": 21}}, \"opc\": {\"pitch_nm\": 1.0, \"guard_band_nm\": 24.0, \"energy_floor\": 0.995}}",
        f);
    std::fclose(f);
  }
  int rc = 0;
  if (litho_image(in.c_str(), cfg.c_str(), (dir + "/capi_aerial.aimg").c_str(), 0.0, 1.0, 0) != LITHO_OK) {
    std::printf("litho_image (aerial) failed: %s\n", litho_last_error());
    rc = 1;
  }
  if (litho_image(in.c_str(), cfg.c_str(), (dir + "/capi_resist.aimg").c_str(), 30.0, 1.1, 1) != LITHO_OK) {
    std::printf("litho_image (resist) failed: %s\n", litho_last_error());
    rc = 1;
  }
  if (litho_ai_init(in.c_str(), cfg.c_str(), (dir + "/capi_ai").c_str()) != LITHO_OK) {
    std::printf("litho_ai_init failed: %s\n", litho_last_error());
    rc = 1;
  }
  if (rc == 0) std::printf("dropin_capi ok\n");
  return rc;
}
