// Engine instantiation for state dimension D = 13.
#define PODE_D 13
#include "inst.cuh"
