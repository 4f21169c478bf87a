// Drop-in forwarding header: code written against the reference's
// "fembatch/oracle.hpp" compiles unchanged against the B200 engine.
#pragma once
#include "../fembatch_b200.hpp"
