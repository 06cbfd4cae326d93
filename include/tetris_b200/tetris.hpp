// Umbrella header of the B200-native drop-in: the reference's
// `#include "tetris/threshold.hpp"` + `using namespace tetris;` becomes
// `#include "tetris_b200/tetris.hpp"` + `using namespace tetris_b200;`.
#pragma once

#include "tetris_b200/core.hpp"
#include "tetris_b200/evaluator.hpp"
#include "tetris_b200/keys.hpp"
#include "tetris_b200/bootstrap.hpp"
