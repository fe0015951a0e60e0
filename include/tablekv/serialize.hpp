// tablekv B200 build — canonical table rendering (drop-in for proj/include/tablekv/serialize.hpp).
#pragma once

#include <string>

#include "tablekv/schema.hpp"

namespace tablekv {

// "table <name>\n" then per column "col <name>[: <desc>][ [pk]][ [fk #<t>.<c>]...]\n".
std::string serialize_table(const TableSchema& schema);

}  // namespace tablekv
