// TEST INFRASTRUCTURE: writes the SSB fixture database (tests/golden/fixture.json)
// with the reference's OWN save_database (/root/reference/proj/src/column_io.cpp,
// compiled in place by make_crys_golden.sh) into tests/golden/crys_fixture/, plus
// three malformed files for the loader's error paths.  Committed output pins
// the B200 CRYS loader (crys_db_load_column_file) to the reference format.
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>

#include "json.hpp"
#include "tq/column_io.hpp"

using namespace tq;
using nlohmann::json;

int main(int argc, char** argv) {
  const std::string fixture = argv[1], out = argv[2];
  std::ifstream in(fixture);
  json j;
  in >> j;
  SsbDatabase db;
  db.scale_factor = 1;
  db.seed = 42;
  for (SsbTable* t : {&db.lineorder, &db.date, &db.supplier, &db.customer, &db.part}) {
    const std::string name = t == &db.lineorder ? "lineorder"
                             : t == &db.date     ? "date"
                             : t == &db.supplier ? "supplier"
                             : t == &db.customer ? "customer"
                                                 : "part";
    t->name = name;
    for (auto& [col, vals] : j["tables"][name].items())
      t->columns.push_back(Column::int32(col, vals.get<std::vector<i32>>()));
  }
  save_database(db, out);
  // a float column and error fixtures next to the database
  save_column(Column::float32("f", {1.5f, -2.25f, 3.0f}), out + "/../crys_float.col");
  {
    std::ofstream b(out + "/../crys_badmagic.col", std::ios::binary);
    b << "CRYZ";
    for (int i = 0; i < 12; ++i) b.put(0);
  }
  {
    std::ofstream b(out + "/../crys_truncated.col", std::ios::binary);
    const unsigned char h[16] = {'C', 'R', 'Y', 'S', 1, 0, 0, 0, 10, 0, 0, 0, 0, 0, 0, 0};
    b.write((const char*)h, 16);
    const int x = 7;
    b.write((const char*)&x, 4);  // 1 of 10 promised elements
  }
  std::printf("wrote %s\n", out.c_str());
  return 0;
}
