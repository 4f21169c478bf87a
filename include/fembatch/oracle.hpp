// Drop-in forwarding header: code written against the reference's
// "fembatch/oracle.hpp" compiles unchanged against the B200 engine (the
// runner / verification modules live in the compatibility library).
#pragma once
#include "../fembatch_compat.hpp"
