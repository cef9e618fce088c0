// Engine instantiation for state dimension D = 11.
#define PODE_D 11
#include "inst.cuh"
