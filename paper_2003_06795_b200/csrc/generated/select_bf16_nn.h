#ifndef SELECT_BF16_NN_H
#define SELECT_BF16_NN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_bf16_nn_config;

static inline select_bf16_nn_config select_bf16_nn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(8870)) {
        if (n < INT64_C(1012)) {
            if (m < INT64_C(4435)) {
                if (k < INT64_C(79)) {
                    if (m < INT64_C(2218)) {
                        if (m < INT64_C(555)) {
                            if (m < INT64_C(278)) {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(28)) {
                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(272)) {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(3072)) {
                        if (n < INT64_C(744)) {
                            if (k < INT64_C(992)) {
                                if (k < INT64_C(167)) {
                                    if (m < INT64_C(555)) {
                                        if (m < INT64_C(159)) {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(278)) {
                                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (k < INT64_C(136)) {
                                            if (m < INT64_C(2218)) {
                                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(111)) {
                                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(2218)) {
                                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (n < INT64_C(203)) {
                                        if (m < INT64_C(70)) {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(744)) {
                                                if (n < INT64_C(144)) {
                                                    if (n < INT64_C(79)) {
                                                        if (m < INT64_C(278)) {
                                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            if (m < INT64_C(1109)) {
                                                                if (m < INT64_C(555)) {
                                                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                                    return out;
                                                                } else {
                                                                    if (k < INT64_C(272)) {
                                                                        if (n < INT64_C(46)) {
                                                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                                            return out;
                                                                        } else {
                                                                            select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                                            return out;
                                                                        }
                                                                    } else {
                                                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                                        return out;
                                                                    }
                                                                }
                                                            } else {
                                                                if (n < INT64_C(46)) {
                                                                    if (m < INT64_C(2218)) {
                                                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                                        return out;
                                                                    } else {
                                                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                                        return out;
                                                                    }
                                                                } else {
                                                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                                    return out;
                                                                }
                                                            }
                                                        }
                                                    } else {
                                                        if (m < INT64_C(555)) {
                                                            if (m < INT64_C(278)) {
                                                                if (k < INT64_C(471)) {
                                                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                                    return out;
                                                                } else {
                                                                    select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                                    return out;
                                                                }
                                                            } else {
                                                                if (k < INT64_C(471)) {
                                                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                                    return out;
                                                                } else {
                                                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                                    return out;
                                                                }
                                                            }
                                                        } else {
                                                            if (k < INT64_C(444)) {
                                                                if (m < INT64_C(1109)) {
                                                                    select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                                    return out;
                                                                } else {
                                                                    if (m < INT64_C(2218)) {
                                                                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                                        return out;
                                                                    } else {
                                                                        if (k < INT64_C(314)) {
                                                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                                            return out;
                                                                        } else {
                                                                            select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                                            return out;
                                                                        }
                                                                    }
                                                                }
                                                            } else {
                                                                if (m < INT64_C(2218)) {
                                                                    if (m < INT64_C(1109)) {
                                                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                                        return out;
                                                                    } else {
                                                                        if (k < INT64_C(544)) {
                                                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                                            return out;
                                                                        } else {
                                                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                                            return out;
                                                                        }
                                                                    }
                                                                } else {
                                                                    select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                                    return out;
                                                                }
                                                            }
                                                        }
                                                    }
                                                } else {
                                                    if (m < INT64_C(139)) {
                                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (m < INT64_C(278)) {
                                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            } else {
                                                if (m < INT64_C(393)) {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(634)) {
                                            if (m < INT64_C(70)) {
                                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (m < INT64_C(1109)) {
                                                if (k < INT64_C(702)) {
                                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (m < INT64_C(2218)) {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(363)) {
                                                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (k < INT64_C(1087)) {
                                    if (m < INT64_C(2218)) {
                                        if (n < INT64_C(363)) {
                                            if (m < INT64_C(278)) {
                                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(555)) {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(1109)) {
                                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(139)) {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(278)) {
                                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (n < INT64_C(363)) {
                                        if (m < INT64_C(2218)) {
                                            if (k < INT64_C(1630)) {
                                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(393)) {
                                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(1630)) {
                                                if (n < INT64_C(182)) {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(2218)) {
                                            if (m < INT64_C(393)) {
                                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(1109)) {
                                                    if (k < INT64_C(2173)) {
                                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(6)) {
                                if (m < INT64_C(3)) {
                                    if (m < INT64_C(2)) {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(29)) {
                                    if (m < INT64_C(12)) {
                                        if (k < INT64_C(1620)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(70)) {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(196)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(555)) {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(3)) {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(70)) {
                                if (m < INT64_C(8)) {
                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(29)) {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(278)) {
                                    if (m < INT64_C(139)) {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            } else {
                if (n < INT64_C(222)) {
                    if (k < INT64_C(118)) {
                        if (k < INT64_C(56)) {
                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(363)) {
                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(544)) {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(3259)) {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        } else {
            if (m < INT64_C(1268)) {
                if (n < INT64_C(1145)) {
                    if (k < INT64_C(363)) {
                        if (m < INT64_C(278)) {
                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (k < INT64_C(10138)) {
                        if (m < INT64_C(12)) {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(139)) {
                                if (k < INT64_C(405)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    if (m < INT64_C(29)) {
                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(70)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(725)) {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(278)) {
                                    if (k < INT64_C(725)) {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(555)) {
                                        if (k < INT64_C(573)) {
                                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (m < INT64_C(3584)) {
                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                    return out;
                }
            }
        }
    } else {
        if (k < INT64_C(815)) {
            if (n < INT64_C(46)) {
                if (k < INT64_C(68)) {
                    if (m < INT64_C(35480)) {
                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(141920)) {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(30)) {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(35480)) {
                        if (k < INT64_C(167)) {
                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                            return out;
                        }
                    } else {
                        select_bf16_nn_config out = {1u, 1u, 1u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                if (k < INT64_C(138)) {
                    if (m < INT64_C(17740)) {
                        if (n < INT64_C(96)) {
                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (k < INT64_C(363)) {
                        if (m < INT64_C(35480)) {
                            if (n < INT64_C(257)) {
                                if (m < INT64_C(17740)) {
                                    if (k < INT64_C(194)) {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(91)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(194)) {
                                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(70960)) {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(91)) {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                }
            }
        } else {
            if (m < INT64_C(35480)) {
                if (n < INT64_C(363)) {
                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                    return out;
                }
            } else {
                select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_BF16_NN_H */
