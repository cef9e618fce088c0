// Engine instantiation for state dimension D = 5.
#define PODE_D 5
#include "inst.cuh"
